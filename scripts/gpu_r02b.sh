#!/bin/bash
# r02 session-2 pass: full -m gpu suite, smoke, default bench, C2b bench, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 2500 gpurun_out/bench_default.json
timeout 600 python bench.py --workload c2b_flux64_s16 --no-cpu-baseline > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err
python scripts/show_bench.py gpurun_out/bench_c2b.json 2>/dev/null | tail -3
