#!/bin/bash
# double-buffered Q (GNA_QBUF=2, 3-slot ring) re-checked on this build; E4M3 with fewer polynomial exps (1/16, none)
O=gpurun_out/ab19; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
GNA_LIB_PATH=$V/libgna_qbuf2.so timeout 120 python scripts/dbg_small.py > $O/dbg_qbuf2.log 2>&1 || { echo "SMOKE qbuf2 FAILED"; cat $O/dbg_qbuf2.log; }
AB_REPS=2 timeout 1500 python scripts/ab.py run c2b_flux64_s16,c4a_hunyuan_blocked,c2a_flux64_s8 base qbuf2 2>&1 | tee $O/ab_qbuf.txt
AB_REPS=2 AB_ARGS="--dtype fp8" timeout 1200 python scripts/ab.py run c4a_hunyuan_blocked base f8poly16 f8poly0 2>&1 | tee $O/ab_f8.txt
