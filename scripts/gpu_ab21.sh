#!/bin/bash
# select-free polynomial exp (GNA_POLY_SCALE) on top of dense-fold + E4M3 poly 1/16: GPU suite and A/B
O=gpurun_out/ab21; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
GNA_LIB_PATH=$V/libgna_next2.so timeout 120 python scripts/dbg_small.py > $O/dbg_next2.log 2>&1 || { echo "SMOKE next2 FAILED"; cat $O/dbg_next2.log; exit 1; }
GNA_LIB_PATH=$V/libgna_next2.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_next2.log 2>&1; tail -2 $O/pytest_next2.log
AB_REPS=3 timeout 2400 python scripts/ab.py run c4a_hunyuan_blocked,x1_hunyuan_s16,c2a_flux64_s8 next next2 2>&1 | tee $O/ab.txt
