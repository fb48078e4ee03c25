#!/bin/bash
# A/B: speculative row max (GNA_SPEC_MAX), with and without split O staging; item timelines base vs split staging
O=gpurun_out/ab14; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
for n in specmax both; do
  GNA_LIB_PATH=$V/libgna_$n.so timeout 120 python scripts/dbg_small.py > $O/dbg_$n.log 2>&1 || { echo "SMOKE $n FAILED"; cat $O/dbg_$n.log; }
done
GNA_LIB_PATH=$V/libgna_specmax.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_fp16.py tests/test_gpu_fullsize.py tests/test_gpu_fp8.py -m gpu -x -q > $O/pytest_specmax.log 2>&1; tail -2 $O/pytest_specmax.log
AB_REPS=2 timeout 1800 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16,c4b_hunyuan_na base specmax both 2>&1 | tee $O/ab.txt
TRACE_LIB=$V/libgna_trace_base.so timeout 300 python scripts/item_timeline.py c2b_flux64_s16 3 > $O/tl_base.txt 2>&1
TRACE_LIB=$V/libgna_trace_ost.so timeout 300 python scripts/item_timeline.py c2b_flux64_s16 3 > $O/tl_ost.txt 2>&1
head -30 $O/tl_base.txt; head -30 $O/tl_ost.txt
