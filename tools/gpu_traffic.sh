cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
export BENCH_NO_CLOCKS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_predict -c 13 -o gpurun_out/traffic_cf python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_tcf.log 2>&1; echo cf rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tma -c 8 -o gpurun_out/traffic_spmm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_tsp.log 2>&1; echo spmm rc=$?
