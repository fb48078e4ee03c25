#!/bin/bash
# P handed to the MMA in 4 chunks instead of 2, re-checked on the final build
O=gpurun_out/ab24; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
GNA_LIB_PATH=$V/libgna_psplit4.so timeout 120 python scripts/dbg_small.py > $O/dbg_psplit4.log 2>&1 || { echo "SMOKE psplit4 FAILED"; cat $O/dbg_psplit4.log; exit 1; }
GNA_LIB_PATH=$V/libgna_psplit4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest_psplit4.log 2>&1; tail -1 $O/pytest_psplit4.log
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,x1_hunyuan_s16,c2b_flux64_s16 base psplit4 2>&1 | tee $O/ab.txt
