#!/bin/bash
# compute-sanitizer over the small-mesh GPU tests (edge tiles incl. the
# multi-sub-bucket path, fans / fallbacks, fused levels, CN TMA ring + tail,
# radix sort, emulated-rank dist kernels, verification).  One log per tool.
# usage (under gpurun, repo root): bash tools/sanitize.sh tag
tag=${1:-r2}
mkdir -p gpurun_out
sel="tests/test_gpu_parity.py tests/test_eg_subbuckets.py tests/test_sparse_ops.py tests/test_dist.py tests/test_verify.py"
kx="not L9 and not large and not 3000 and not config1 and not config4 and not config2 and not permuted_node"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
     python -m pytest $sel -m gpu -x -q -k "$kx" -p no:cacheprovider > gpurun_out/sanitize_${tool}_$tag.log 2>&1
  echo "exit $? ($tool)" >> gpurun_out/sanitize_${tool}_$tag.log
  tail -4 gpurun_out/sanitize_${tool}_$tag.log
done
