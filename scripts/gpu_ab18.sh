#!/bin/bash
# E4M3 kernel: polynomial exp share 1/8 (default) vs 1/4, 1/3, 1/2 (half the tensor time per exp: MUFU-bound)
O=gpurun_out/ab18; mkdir -p $O
V=$PWD/paper_2504_16922_b200/variants
GNA_LIB_PATH=$V/libgna_f8poly4.so timeout 600 python -m pytest tests/test_gpu_fp8.py -m gpu -x -q > $O/pytest_f8poly4.log 2>&1; tail -1 $O/pytest_f8poly4.log
AB_REPS=2 AB_ARGS="--dtype fp8" timeout 2400 python scripts/ab.py run c4a_hunyuan_blocked,c2b_flux64_s16 base f8poly4 f8poly3 f8poly2 2>&1 | tee $O/ab.txt
