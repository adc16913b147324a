# A/B of library variants on the headline step and the given-L13 line
for v in default "$@" default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2401_15557_b200/variants/libphfem_b200_$v.so; fi
  PHFEM_LIB=$lib timeout 600 python bench.py --no-cpu --no-e2e --no-cn --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); ms=d['ms_per_step']; sh=d['kernel_share']
print('$v', round(ms,3), 'given', round(d['config5_given_mesh']['ms_per_step'],3), {k: round(sh.get(k,0)*ms,3) for k in ('k_eg_emit','k_eg_tile')})"
done
