#!/bin/bash
# ncu --set full of the attention kernel (last of 2 launches) per workload; DRAM bytes per launch
# -> gpurun_out/ncu_<wl>_<dt>.ncu-rep (summarised here by scripts/ncu_traffic.py)
mkdir -p gpurun_out
for spec in ${NCU_SPECS:-c4a_hunyuan_blocked:bf16 c2b_flux64_s16:bf16}; do
  wl=${spec%%:*}; dt=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gna_attn --launch-skip 1 --launch-count 1 \
      -f -o gpurun_out/ncu_${wl}_${dt} python scripts/one_launch.py $wl $dt 2 > gpurun_out/ncu_${wl}_${dt}.log 2>&1
  echo "$spec rc=$?"
done
