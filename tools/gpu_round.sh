#!/bin/bash
# Round measurement in one gpurun call: GPU suite, smoke, bench (all lines),
# reference arm, launch list of the L13 step, ncu --set full of the step's
# top kernels.   usage (repo root, under gpurun): bash tools/gpu_round.sh tag
tag=${1:-r2}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$tag.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench exit $?" >> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference > gpurun_out/ref_arm_$tag.json 2> gpurun_out/ref_arm_$tag.err
timeout 600 python tools/profile_step.py 13 > gpurun_out/plain_$tag.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/profile_step.py 13 > gpurun_out/ncu_launch_$tag.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch_$tag.log
# the L12 input build launches 12 x (k_eg_tile_col + k_eg_emit); the step's
# five heaviest kernels follow
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:k_eg_tile_col|k_rl_level|k_volume|k_refine_children|k_eg_emit' \
   -s 24 -c 5 -o gpurun_out/prof_step_$tag python tools/profile_step.py 13 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full_$tag.log
# the report can exceed what gpurun brings back: summarise it on the box
python tools/ncu_summary.py gpurun_out/prof_step_$tag.ncu-rep > gpurun_out/ncu_full_L13_step_$tag.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_step_$tag.ncu-rep k_volume 30 > gpurun_out/ncu_sass_k_volume_$tag.txt 2>&1
for f in pytest_gpu_$tag.log smoke_$tag.log bench_$tag.err ncu_launch_$tag.log ncu_full_$tag.log; do tail -n 3 gpurun_out/$f; done
