#!/bin/bash
V=paper_2504_16922_b200/variants
timeout 120 python scripts/dbg_small.py > /dev/null 2>&1 || { echo "SMOKE base FAILED"; exit 1; }
GNA_LIB_PATH=$V/libgna_eo.so timeout 120 python scripts/dbg_small.py 2>&1 | tail -2; [ ${PIPESTATUS[0]} -eq 0 ] || { echo "SMOKE eo FAILED"; exit 1; }
GNA_LIB_PATH=$V/libgna_eo.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_fp8.py -m gpu -x -q 2>&1 | tail -2
TRACE_LIB=$V/libgna_t_eo.so timeout 300 python scripts/item_timeline.py c2b_flux64_s16 1 2>&1 | grep -v warning | tail -9
AB_REPS=2 timeout 1500 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base eo ns3
