mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_select.py > gpurun_out/probe_select.txt 2>&1
timeout 600 python bench.py --no-cpu --no-explore --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
