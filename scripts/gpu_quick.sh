#!/bin/bash
# quick GPU pass: build, a parity subset, persistent vs one-CTA-per-item bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_fp8.py tests/test_gpu_fp16.py -m gpu -x -q -rf ${PYTEST_ARGS} > gpurun_out/pytest_quick.log 2>&1
tail -3 gpurun_out/pytest_quick.log
for wl in c4a_hunyuan_blocked c2b_flux64_s16 c4b_hunyuan_na; do
  for ps in 1 0; do
    GNA_PERSIST=$ps timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-verify > gpurun_out/q_${wl}_p$ps.json 2>gpurun_out/q_${wl}_p$ps.err
    python -c "import json;d=json.loads(open('gpurun_out/q_${wl}_p$ps.json').read().strip().splitlines()[-1]);print('$wl persist=$ps', round(d['value'],1), 'TF/s', d['clocks']['sm_mhz'], 'MHz', round(d['value']/d['clocks']['sm_mhz']*1000,1), '/GHz', 'speedup', round(d['speedup_vs_dense'],3), 'bound', round(d['bound'],3))" 2>&1 | tail -1
  done
done
