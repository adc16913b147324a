#!/bin/bash
# bench (all lines), given-L13 per-kernel profile, config-4 sector metrics,
# ncu --set full of the given-L13 edge tile + emit passes.
tag=${1:-r2c}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench exit $?" >> gpurun_out/bench_$tag.err
timeout 300 python tools/profile_given.py 13 > gpurun_out/given_$tag.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum
timeout 900 ncu --nvtx --nvtx-include "c4step/" --metrics $M --clock-control none --csv \
   --log-file gpurun_out/config4_sectors_$tag.csv python tools/profile_config4.py 12 > gpurun_out/config4_ncu_$tag.log 2>&1
echo "ncu c4 exit $?" >> gpurun_out/config4_ncu_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_eg_tile$|k_eg_emit' -s 26 -c 2 \
   -o gpurun_out/prof_given_$tag python tools/profile_given.py 13 --once > gpurun_out/ncu_given_$tag.log 2>&1
echo "ncu given exit $?" >> gpurun_out/ncu_given_$tag.log
tail -2 gpurun_out/bench_$tag.err; cat gpurun_out/given_$tag.txt; tail -2 gpurun_out/config4_ncu_$tag.log gpurun_out/ncu_given_$tag.log
