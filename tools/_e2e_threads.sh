# e2e sweep: host threads / direct-chunk split of the download (one gpurun call)
for k in 0 3 2 4 3 0; do
  PHFEM_DL_DIRECT_EVERY=$k timeout 600 python bench.py --no-cpu --no-cn --no-given --steps 3 --e2e-steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('direct_every $k', round(e['value']/1e6,1), 'Mtri/s', round(e['ms_per_step'],1), 'ms', 'wire', e['d2h_bytes_per_step'])"
done
