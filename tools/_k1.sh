#!/bin/bash
# K1 iteration: draft/selector parity tests, selector phase probe, ncu source page of K1 at 16M.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "draft or fused or config3 or full_size or round_matches or population or division" > gpurun_out/pytest_k1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k1.log
timeout 300 python tools/probe_select.py round > gpurun_out/probe_select_round.txt 2>&1
bash tools/_ncu1.sh k_fsel kfsel16m gemm1024 16777216 fp64 3
