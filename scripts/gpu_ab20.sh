#!/bin/bash
# dense-item flag folded into a stage count (no per-stage local load) + E4M3 polynomial share 1/16: GPU suite and A/B
O=gpurun_out/ab20; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
GNA_LIB_PATH=$V/libgna_next.so timeout 120 python scripts/dbg_small.py > $O/dbg_next.log 2>&1 || { echo "SMOKE next FAILED"; cat $O/dbg_next.log; exit 1; }
GNA_LIB_PATH=$V/libgna_next.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_next.log 2>&1; tail -2 $O/pytest_next.log
AB_REPS=2 timeout 2400 python scripts/ab.py run c4a_hunyuan_blocked,c3_cosmos,x2_flux4k,c2b_flux64_s16 base densefold next 2>&1 | tee $O/ab.txt
