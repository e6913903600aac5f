# timed-step outliers by clock sampler: nvml (in-process) vs smi (nvidia-smi -lms)
cd $GRAFT_REPO_ROOT
for i in 1 2 3 4 5 6 7 8; do
  for mode in nvml; do
    BENCH_CLOCKS=$mode python bench.py --no-cpu-baseline --no-variants --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); st=d['step_times_s']; print('$mode', d['ms_per_step'], d['allocator_in_timed_region'], [ (i, round(x*1e3,1)) for i,x in enumerate(st) if x > 0.0435])"
  done
done
