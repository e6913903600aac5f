cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
export BENCH_NO_CLOCKS=1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/b_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_l.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_predict|k_spmm_pipe" -s 30 -c 4 -o gpurun_out/top python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-variants > gpurun_out/ncu_top.log 2>&1; echo full rc=$?
