for v in eg_nolb eg_v2 eg_v8; do
  PHFEM_LIB=paper_2401_15557_b200/variants/libphfem_b200_$v.so timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/var_base.json 2> gpurun_out/var_base.err
