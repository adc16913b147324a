"""Summarise an ncu report: key raw metrics per kernel + top stall SASS lines.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex-for-sass]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'lts__t_sector_hit_rate.pct',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
ki = hdr.index('Kernel Name')
for r in rows[2:]:
    print('=====', r[ki][:90])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f'  {w:80s} {r[i]} {units[i]}')
if len(sys.argv) > 2:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                          '--kernel-name', 'regex:' + sys.argv[2]], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
    hdr, data = rows[hi], rows[hi + 1:]
    # several kernels in one report: keep the first kernel's table
    end = next((i for i, r in enumerate(data) if r and r[0] in ('Kernel Name', 'Address')), len(data))
    data = data[:end]
    si = hdr.index('Warp Stall Sampling (All Samples)')
    ie = hdr.index('Instructions Executed')
    tot = sum(float(r[si] or 0) for r in data) or 1
    top = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
    for i in sorted(top):
        r = data[i]
        print(f"{i:5d} {float(r[si]) / tot * 100:5.1f}% ie={r[ie]:>10} {r[1][:90]}")
