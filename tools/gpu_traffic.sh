#!/bin/bash
# ncu --set full captures of the two roofline kernels over one bench step
# (every CF scoring launch, 8 SpMM launches) -> gpurun_out/traffic_*.ncu-rep;
# tools/traffic.py turns them into profiles/traffic.json.
cd "${GRAFT_REPO_ROOT:-.}"
export BENCH_NO_CLOCKS=1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_predict -c 13 -o gpurun_out/traffic_cf python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_tcf.log 2>&1; echo cf rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_pipe -c 8 -o gpurun_out/traffic_spmm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_tsp.log 2>&1; echo spmm rc=$?
