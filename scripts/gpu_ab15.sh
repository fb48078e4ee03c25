#!/bin/bash
# masked-stage diet (host comb constants, per-half mask skip) + 32-bit item counters: GPU suite and A/B vs HEAD
O=gpurun_out/ab15; mkdir -p $O
timeout 120 python scripts/dbg_small.py > $O/dbg_base.log 2>&1 || { echo "SMOKE base FAILED"; cat $O/dbg_base.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
AB_REPS=2 timeout 2400 python scripts/ab.py run c2a_flux64_s8,c4b_hunyuan_na,s2c_sweep2d_causal,c4a_hunyuan_blocked,c3_cosmos head base 2>&1 | tee $O/ab.txt
