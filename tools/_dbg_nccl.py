import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import torch.distributed as tdist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29518")
torch.cuda.set_device(0)
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from oracle import oracle as O
from paper_2401_15557_b200 import capi, dist, meshgen as G
dev = torch.device("cuda", 0)
ctx = capi.Context(0, stream=torch.cuda.current_stream(dev).cuda_stream)
for lv in (9, 11, 12):
    from bench import build_input
    hm = build_input(ctx, lv).download()
    comm = dist.TorchComm()
    states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(ctx, dev))
    s = states[0]
    splits = np.asarray([0, hm.nC], np.int32)
    send, cnt = s.ops.occurrences(s.elements, s.elo, s.ehi, s.ops.as_tensor(splits), pack=True)
    print("lv", lv, "send", tuple(send.shape), "cnt", cnt, "nE", hm.nE, flush=True)
    try:
        st, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *G.config_fields(5))
        print("ok", nC, nE, st[0].stats)
    except Exception as e:
        print("ERR", e)
tdist.destroy_process_group()
