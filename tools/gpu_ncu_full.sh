#!/bin/bash
# One gpurun call: ncu --set full capture of the step's three heaviest kernels
# (L11 -> L12 step: k_eg_tile of the parent build, k_rl_emit<1>, k_volume).
# usage: bash tools/gpu_ncu_full.sh tag [level]
tag=${1:-r1}; lvl=${2:-12}
mkdir -p gpurun_out
skip=$((lvl - 1))
timeout 600 python tools/profile_step.py $lvl > gpurun_out/plain_full_$tag.log 2>&1 &&
timeout 1800 ncu --set full --clock-control none --import-source on \
   -k regex:'k_eg_tile$|k_rl_emit|k_volume' -s $skip -c 3 -o gpurun_out/prof_$tag \
   python tools/profile_step.py $lvl > gpurun_out/ncu_full_$tag.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_$tag.log
tail -5 gpurun_out/ncu_full_$tag.log
