#!/bin/bash
# last pass of round 2 (64-bit item counters restored): GPU suite, smoke, default / fp16 / E4M3 bench lines, launch list
O=gpurun_out/final3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 python scripts/dbg_small.py > $O/dbg_small.log 2>&1 || { echo "SMOKE FAILED"; cat $O/dbg_small.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --dtype fp16 --no-cpu-baseline > $O/bench_fp16_c4a.json 2> $O/bench_fp16_c4a.err
timeout 600 python bench.py --dtype fp8 --no-cpu-baseline > $O/bench_fp8_c4a.json 2> $O/bench_fp8_c4a.err
timeout 600 python bench.py --workload x1_hunyuan_s16 --no-cpu-baseline > $O/bench_x1_hunyuan_s16.json 2> $O/bench_x1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-verify > $O/ncu_launch_bench.log 2>&1
for f in $O/bench_*.json; do python scripts/show_bench.py $f 2>/dev/null | cut -c1-200; done
