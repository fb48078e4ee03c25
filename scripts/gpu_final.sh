#!/bin/bash
# round-2 final pass: build, GPU suite, smoke, ncu traffic captures (their summary feeds the bench lines'
# roofline.traffic), bench lines (default + workloads + dtypes + reference), launch list of the default command
O=${OUT:-gpurun_out/final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 python scripts/dbg_small.py > $O/dbg_small.log 2>&1 || { echo "SMOKE FAILED"; cat $O/dbg_small.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
NCU_SPECS="c4a_hunyuan_blocked:bf16 c2b_flux64_s16:bf16 c2a_flux64_s8:bf16" bash scripts/ncu_traffic.sh
python scripts/ncu_traffic.py gpurun_out/ncu_c4a_hunyuan_blocked_bf16.ncu-rep gpurun_out/ncu_c2b_flux64_s16_bf16.ncu-rep gpurun_out/ncu_c2a_flux64_s8_bf16.ncu-rep > $O/ncu_traffic.log 2>&1
cp profiles/r02_ncu_traffic.json $O/r02_ncu_traffic.json
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for wl in c2b_flux64_s16 c3_cosmos x1_hunyuan_s16 x2_flux4k x3_cosmos89 c4b_hunyuan_na c2a_flux64_s8 s2c_sweep2d_causal s3_sweep3d; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 600 python bench.py --dtype fp16 --no-cpu-baseline > $O/bench_fp16_c4a.json 2> $O/bench_fp16_c4a.err
timeout 600 python bench.py --dtype fp8 --no-cpu-baseline > $O/bench_fp8_c4a.json 2> $O/bench_fp8_c4a.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-verify > $O/ncu_launch_bench.log 2>&1
for f in $O/bench_*.json; do python scripts/show_bench.py $f 2>/dev/null | cut -c1-200; done
