for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2401_15557_b200/variants/libphfem_b200_$v.so; fi
  PHFEM_LIB=$lib timeout 600 python bench.py --no-cpu --no-e2e --no-cn --no-given --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/var_{sys.argv[1]}.json"))
ms = d["ms_per_step"]; sh = d["kernel_share"]
print(sys.argv[1], round(ms, 3), {k: round(sh[k] * ms, 3) for k in ("k_volume", "k_rl_level_full", "k_refine_children")})
PY
done
