import os, sys, json
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi
class A: cn_level = 11
ctx = capi.Context(0)
print(os.environ.get("PHFEM_LIB", "default"), json.dumps(bench.run_cn_rhs(ctx, A())))
