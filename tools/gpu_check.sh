#!/bin/bash
# One GPU session: parity tests, smoke, bench (fp64 default + bf16), ncu launch list, GA explore bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --precision bf16 --no-cpu > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-explore > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/explore_bench.py --reps 20 > gpurun_out/explore.log 2>&1
echo done
