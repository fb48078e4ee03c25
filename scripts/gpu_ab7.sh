#!/bin/bash
V=paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py > /dev/null 2>&1 || { echo "SMOKE base FAILED"; exit 1; }
GNA_LIB_PATH=$V/libgna_mma2.so timeout 120 python scripts/dbg_small.py 2>&1 | tail -3 || { echo "SMOKE mma2 FAILED"; exit 1; }
GNA_LIB_PATH=$V/libgna_mma2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fp16.py tests/test_gpu_fp8.py -m gpu -x -q 2>&1 | tail -2
for t in t_base t_mma2; do
  echo "== $t"; TRACE_LIB=$V/libgna_$t.so timeout 200 python scripts/trace_attn.py c4a_hunyuan_blocked 2>&1 | grep -A1 "chunk0" | head -2
done
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base mma2
