# one gpurun call: the L13 step with the default library and each variant
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2401_15557_b200/variants/libphfem_b200_$v.so; fi
  PHFEM_LIB=$lib timeout 600 python bench.py --no-cpu --no-e2e --no-cn --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/var_{sys.argv[1]}.json"))
kr = d["kernel_roofline"]
print(sys.argv[1], round(d["ms_per_step"], 3), {k: v["ms"] for k, v in list(kr.items())[:5]})
PY
done
