#!/bin/bash
# softmax-structure A/B: parity (base + all3), cycle traces per variant, bench A/B
V=paper_2504_16922_b200/variants
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
GNA_LIB_PATH=$V/libgna_all3p4.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for t in t_base t_sumlate t_defer8 t_ldsplit t_all3 t_all3p4; do
  echo "== $t"; TRACE_LIB=$V/libgna_$t.so timeout 300 python scripts/trace_attn.py c4a_hunyuan_blocked 2>&1 | grep -A1 "chunk0" | head -2
done
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base sumlate defer8 ldsplit all3 all3p4
