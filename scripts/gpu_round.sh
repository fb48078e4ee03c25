#!/bin/bash
# bench (default C4a + C2b + fp16) + sanitizer + the two ABI tests that failed
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_abi.py -q -rf > gpurun_out/pytest_abi.log 2>&1; tail -2 gpurun_out/pytest_abi.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
timeout 600 python bench.py --workload c2b_flux64_s16 --no-cpu-baseline > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err
timeout 600 python bench.py --dtype fp16 --no-cpu-baseline > gpurun_out/bench_fp16.json 2> gpurun_out/bench_fp16.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash scripts/gpu_sanitize.sh
