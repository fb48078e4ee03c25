#!/bin/bash
# separate the two changes of ab15: mask diet alone, 32-bit item counters alone
O=gpurun_out/ab16; mkdir -p $O
AB_REPS=2 timeout 2400 python scripts/ab.py run c4a_hunyuan_blocked,c3_cosmos,c2a_flux64_s8 head base maskonly intonly 2>&1 | tee $O/ab.txt
