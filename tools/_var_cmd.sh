bash tools/gpu_check.sh r1m
for v in egm; do
  PHFEM_LIB=paper_2401_15557_b200/variants/libphfem_b200_$v.so timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
