#!/bin/bash
# 32-bit item counters (default since the mask-diet commit) vs 64-bit, bf16 and E4M3 C4a
O=gpurun_out/ab23; mkdir -p $O
AB_REPS=3 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked base ll 2>&1 | tee $O/ab_bf16.txt
AB_REPS=3 AB_ARGS="--dtype fp8" timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked base ll 2>&1 | tee $O/ab_fp8.txt
