#!/bin/bash
# Round-end evidence on one GPU: parity suite, smoke, bench (both arms), config-5 sweep,
# selector phase probe, launch list of the bench, ncu --set full of K1 at 16M.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 900 python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
timeout 300 python tools/probe_select.py round > gpurun_out/probe_select_round.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-explore --no-bert > gpurun_out/ncu_bench.log 2>&1
bash tools/_ncu1.sh k_fsel kfsel16m gemm1024 16777216 fp64 3
echo done
