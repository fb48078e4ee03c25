#!/bin/bash
# bf16/fp16 polynomial exp share with the select-free polynomial: 1/8 (default) vs 1/4, 1/6, 1/16
O=gpurun_out/ab22; mkdir -p $O
AB_REPS=2 timeout 2400 python scripts/ab.py run c4a_hunyuan_blocked,x1_hunyuan_s16,c2b_flux64_s16 base poly4 poly6 poly16 2>&1 | tee $O/ab.txt
