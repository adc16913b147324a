# given-L13 step per library variant (tools/_given13.py)
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2401_15557_b200/variants/libphfem_b200_$v.so; fi
  echo "== $v"; PHFEM_LIB=$lib timeout 600 python tools/_given13.py 2>&1 | head -5
done
