#!/bin/bash
# 64-bit row mask for 64-token boxes (in-tree build) vs the 128-bit form (maskdiet) vs HEAD; GPU suite of the in-tree build
O=gpurun_out/ab17; mkdir -p $O
timeout 120 python scripts/dbg_small.py > $O/dbg_base.log 2>&1 || { echo "SMOKE base FAILED"; cat $O/dbg_base.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
AB_REPS=2 timeout 2400 python scripts/ab.py run c2a_flux64_s8,c4b_hunyuan_na,s3_sweep3d,s2c_sweep2d_causal,c4a_hunyuan_blocked head maskdiet base 2>&1 | tee $O/ab.txt
