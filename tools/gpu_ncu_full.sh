#!/bin/bash
# One gpurun call: ncu --set full capture of the step's heaviest kernels.
# usage: bash tools/gpu_ncu_full.sh tag [level] [kernel-regex] [skip] [count]
# (defaults: L11 -> L12 step; k_eg_tile of the parent build, the fused refined
#  level, k_volume; skip = the level-1 k_eg_tile launches of the input build)
tag=${1:-r1}; lvl=${2:-12}
rx=${3:-'k_eg_tile$|k_rl_level|k_volume'}
skip=${4:-$((lvl - 1))}; cnt=${5:-3}
mkdir -p gpurun_out
timeout 600 python tools/profile_step.py $lvl > gpurun_out/plain_full_$tag.log 2>&1 &&
timeout 1800 ncu --set full --clock-control none --import-source on \
   -k "regex:$rx" -s $skip -c $cnt -o gpurun_out/prof_$tag \
   python tools/profile_step.py $lvl > gpurun_out/ncu_full_$tag.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_$tag.log
grep PROF gpurun_out/ncu_full_$tag.log | tail -5
