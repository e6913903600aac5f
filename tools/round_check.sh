#!/bin/bash
# Full GPU validation of the working tree (gpurun): all -m gpu tests, smoke,
# the default bench line, the reference arm and an ncu launch list of a short
# bench (per-launch kernel times), each with its own log under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/rc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rc_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc_smoke.log
timeout 900 python bench.py > gpurun_out/rc_bench.log 2> gpurun_out/rc_bench.err; echo "bench rc=$?" >> gpurun_out/rc_bench.err
if [ -z "$SKIP_REF" ]; then timeout 600 python bench.py --impl reference > gpurun_out/rc_ref.log 2> gpurun_out/rc_ref.err; fi
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/rc_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/rc_ncu.log 2>&1
fi
echo done
