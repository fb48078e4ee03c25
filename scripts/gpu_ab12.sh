#!/bin/bash
V=paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py > /dev/null 2>&1 || { echo "SMOKE base FAILED"; exit 1; }
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base nosusp susp10k
