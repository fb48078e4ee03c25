#!/bin/bash
V=paper_2504_16922_b200/variants
for v in bd1 bd2; do GNA_LIB_PATH=$V/libgna_$v.so timeout 120 python scripts/dbg_small.py > /dev/null 2>&1 || { echo "SMOKE $v FAILED"; exit 1; }; done
for t in t_bd0 t_bd1; do
  echo "== $t"; TRACE_LIB=$V/libgna_$t.so timeout 200 python scripts/trace_attn.py c4a_hunyuan_blocked 2>&1 | grep -A1 "chunk0" | head -2
done
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base bd1 bd2 bd1m88
