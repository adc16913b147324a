#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench exit $?" >> gpurun_out/bench_$tag.err
timeout 600 python tools/profile_step.py 13 > gpurun_out/plain_$tag.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/profile_step.py 13 > gpurun_out/ncu_launch_$tag.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_launch_$tag.log
tail -3 gpurun_out/pytest_gpu_$tag.log gpurun_out/smoke_$tag.log; cat gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
