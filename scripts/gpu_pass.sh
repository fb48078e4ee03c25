#!/bin/bash
# One GPU pass: tests, bench lines, ncu launch list and a full capture of the attention kernel.
# usage: scripts/gpu_pass.sh TAG [tests|bench|ncu|all] [workloads...]
set -u
TAG=${1:-r01}; WHAT=${2:-all}; shift 2 || true
WLS=${@:-c2b_flux64_s16}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [[ $WHAT == tests || $WHAT == all ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -o timeout=120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
fi
if [[ $WHAT == bench || $WHAT == all ]]; then
  for wl in $WLS; do
    timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err; echo "bench $wl rc=$?"; cut -c1-600 $OUT/bench_$wl.json
  done
fi
if [[ $WHAT == fp8 || $WHAT == all ]]; then
  for wl in $WLS; do
    timeout 600 python bench.py --workload $wl --dtype fp8 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_fp8_$wl.json 2> $OUT/bench_fp8_$wl.err; echo "bench fp8 $wl rc=$?"; cut -c1-300 $OUT/bench_fp8_$wl.json
  done
fi
if [[ $WHAT == ncuattn ]]; then
  for wl in $WLS; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:gna_attn -s 3 -c 1 -o $OUT/attn_$wl \
      python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_full_$wl.log 2>&1; echo "ncu full $wl rc=$?"
  done
fi
if [[ $WHAT == ncu || $WHAT == all ]]; then
  for wl in $WLS; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$wl.csv \
      python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list $wl rc=$?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:gna_attn -s 3 -c 1 -o $OUT/attn_$wl \
      python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_full_$wl.log 2>&1; echo "ncu full $wl rc=$?"
    timeout 900 ncu --set full --clock-control none -k regex:permute -s 1 -c 2 -o $OUT/perm_$wl \
      python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_perm_$wl.log 2>&1; echo "ncu perm $wl rc=$?"
  done
fi
