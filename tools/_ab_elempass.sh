# A/B: elem_edge by the element pass (default) vs scattered by the emit pass
for v in 1 0 1 0; do
  PHFEM_EG_ELEMPASS=$v timeout 600 python bench.py --no-cpu --no-e2e --no-cn --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); ms=d['ms_per_step']; sh=d['kernel_share']
print('elempass $v', round(ms,3), 'given', round(d['config5_given_mesh']['ms_per_step'],3), {k: round(sh.get(k,0)*ms,3) for k in ('k_eg_emit','k_eg_elem_edge','k_eg_tile')})"
done
