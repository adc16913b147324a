"""One config-4 step (stress L12 -> normalise -> EG -> RF -> L13 EG + AS) inside
an NVTX range "c4step", for ncu:
  ncu --nvtx --nvtx-include "c4step/" --metrics ... python tools/profile_config4.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import config4_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 12
ctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
dm, keep, nflip = config4_input(ctx, level)
ctx.sync()
torch.cuda.nvtx.range_push("c4step")
capi.orient_ccw(ctx, dm)
capi.pipeline(ctx, dm, 1, *G.config_fields(4)).release()
ctx.sync()
torch.cuda.nvtx.range_pop()
print(f"config4 step ok: L{level} {dm.m.nE} triangles, {nflip} flipped")
