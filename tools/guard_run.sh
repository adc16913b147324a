#!/bin/bash
# The GPU suite under guard mode (red zones + poisoned payloads), twice with
# different poison bytes; logs under gpurun_out/.   usage: bash tools/guard_run.sh tag
tag=${1:-r2}
mkdir -p gpurun_out
for poison in 0xff 0x00; do
  PHFEM_GUARD=1 PHFEM_GUARD_POISON=$poison timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
     > gpurun_out/guard_${poison}_$tag.log 2>&1
  echo "exit $? (PHFEM_GUARD=1 PHFEM_GUARD_POISON=$poison)" >> gpurun_out/guard_${poison}_$tag.log
  tail -3 gpurun_out/guard_${poison}_$tag.log
done
