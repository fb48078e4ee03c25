#!/bin/bash
# A/B: per-warpgroup split O staging with early Q release (GNA_OST_SPLIT) vs the default epilogue
O=gpurun_out/ab13; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py > $O/dbg_base.log 2>&1 || { echo "SMOKE base FAILED"; cat $O/dbg_base.log; exit 1; }
GNA_LIB_PATH=$V/libgna_ostsplit.so timeout 120 python scripts/dbg_small.py > $O/dbg_ostsplit.log 2>&1 || { echo "SMOKE ostsplit FAILED"; cat $O/dbg_ostsplit.log; }
GNA_LIB_PATH=$V/libgna_ostsplit.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_fp16.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest_ostsplit.log 2>&1; tail -2 $O/pytest_ostsplit.log
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16,c3_cosmos base ostsplit 2>&1 | tee $O/ab.txt
