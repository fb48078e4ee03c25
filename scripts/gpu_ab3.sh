#!/bin/bash
# producer-wait sleep A/B (hang-guarded)
V=paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py 2>&1 | tail -3; rc=${PIPESTATUS[0]}
if [ $rc -ne 0 ]; then echo "SMOKE FAILED rc=$rc"; exit 1; fi
for v in earlyq l2m88; do GNA_LIB_PATH=$V/libgna_$v.so timeout 120 python scripts/dbg_small.py > /dev/null 2>&1 || echo "SMOKE $v FAILED"; done
AB_REPS=2 timeout 2000 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base nosleep qonly q1024 kv256 earlyq lag2 l2m88 m88
