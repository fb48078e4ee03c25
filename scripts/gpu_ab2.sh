#!/bin/bash
# quick hang-guarded smoke first; abort the A/B if the default build fails it
V=paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py 2>&1 | tail -7; rc=${PIPESTATUS[0]}
if [ $rc -ne 0 ]; then echo "SMOKE FAILED rc=$rc"; exit 1; fi
GNA_LIB_PATH=$V/libgna_lag3.so timeout 120 python scripts/dbg_small.py 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for t in t_lag0 t_lag2 t_lag3; do
  echo "== $t"; TRACE_LIB=$V/libgna_$t.so timeout 200 python scripts/trace_attn.py c4a_hunyuan_blocked 2>&1 | grep -A1 "chunk0" | head -2
done
AB_REPS=2 timeout 1800 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base lateq0 lag1 lag2 lag3 lag4 lag3p4
