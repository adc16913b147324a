"""Multi-GPU edge generation -> red refinement -> assembly.

One rank per GPU.  Elements are partitioned into contiguous ranges (their
children keep the partition: the children of [a, b) are [4a, 4b),
refine.cpp:28-37); max nodes into contiguous key ranges, so every rank owns a
contiguous range of canonical edge ids.  Per-element work (blocks, load,
children of the own elements) needs no communication.  The exchanges:

  edge dedup     key-range all-to-all of the directed occurrences, a local
                 sort (phfem_dist_dedup: the single-GPU tile kernels), an
                 all-gather of the per-rank edge counts (global ids), and a
                 reverse all-to-all of (element slot, edge id) pairs;
  refinement     midpoints of the owned edges, all-gathered (coordinates stay
                 replicated); boundary lists bisected from the resolved ids;
  boundary data  all-reduce of the boundary-pair ids and of the Neumann edge
                 table (both O(sqrt N)).

The concatenation of the ranks' outputs is bit-identical to the single-GPU
pipeline (tests/test_dist.py): numbering depends only on keys, t_plus only on
element ids.

The orchestration runs phase by phase over the rank states this process
owns: one under torchrun (TorchComm: NCCL on GPUs, gloo on CPU) or W
emulated ranks in one process (LocalComm) — the latter runs the real kernels
of W ranks on one GPU one after another, never concurrently, so no rank ever
waits on another.  Per-rank operations come from a backend: CudaRankOps (the
product: C-ABI kernels); the CPU tests plug in a numpy restatement
(tests/dist_cpu_backend.py) to exercise the exchanges with gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

import numpy as np
import torch

from . import capi

import os as _os
import time as _time


class _Trace:
    """PHFEM_DIST_TRACE=1: synchronising per-phase wall times (debug only)."""

    def __init__(self, states):
        self.on = _os.environ.get("PHFEM_DIST_TRACE") is not None
        self.t = _time.perf_counter()
        self.dev = states[0].coords.device if states else None
        self.rows = []

    def __call__(self, what):
        if not self.on:
            return
        if self.dev is not None and self.dev.type == "cuda":
            torch.cuda.synchronize(self.dev)
        now = _time.perf_counter()
        self.rows.append((what, (now - self.t) * 1e3))
        self.t = now

    def dump(self):
        if self.on:
            print("[dist] " + "  ".join(f"{w}={ms:.2f}" for w, ms in self.rows), flush=True)

NO_ERROR = -1  # int64 view of the uint64 ~0 the kernels start from (all-reduced as unsigned below)


# ---- communication ------------------------------------------------------------------
class TorchComm:
    """torch.distributed: this process is one rank (NCCL on GPUs, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.ranks = [dist.get_rank()]
        self._win = {}
        # the last level's volume pass on a side stream (tested bit-exact;
        # measured at N = 1: 20.96 -> 20.84 ms, 21.18 with a high-priority
        # main stream — the small kernels and NCCL's of the synchronising
        # phases queue behind its CTAs), so off unless asked for
        self.overlap_volume = False

    def all_reduce(self, ts: list, op: str):
        o = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX, "min": self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(ts[0], op=o)

    def all_gather(self, ts: list) -> list:
        out = [torch.empty_like(ts[0]) for _ in range(self.world)]
        self.dist.all_gather(out, ts[0])
        return [out]

    def window(self, ts: list, key: str = "") -> list:
        """Peer window: every rank's tensor mapped into this process (CUDA IPC
        through torch's storage sharing; over NVLink between GPUs).  Returns,
        per local state, the W tensors in rank order.  The mappings are cached
        per key while every rank's buffer stays the same (one all-reduced
        flag decides; opening IPC handles costs milliseconds, so a step must
        not pay it)."""
        t = ts[0]
        if self.world == 1:
            return [[t]]
        st = t.untyped_storage()
        sig = (st.data_ptr(), st.nbytes())
        cached = self._win.get(key)
        need = torch.tensor([0 if cached is not None and cached[0] == sig else 1], dtype=torch.int32,
                            device=t.device)
        self.dist.all_reduce(need, op=self.dist.ReduceOp.MAX)
        if int(need.item()) == 0:
            return [cached[1]]
        from torch.multiprocessing.reductions import reduce_tensor
        objs = [None] * self.world
        self.dist.all_gather_object(objs, reduce_tensor(t))
        me = self.ranks[0]
        views = [t if r == me else fn(*args) for r, (fn, args) in enumerate(objs)]
        self._win[key] = (sig, views)
        return [views]

    def fence(self):
        """every rank's peer stores complete and visible before anyone reads.
        NCCL: a one-element all-reduce on the stream — it completes on a rank
        only after every rank's preceding kernels (the peer stores) finished,
        and orders the reader's next kernels after it, with no host sync.
        Other backends: device synchronise + barrier.  One rank: nothing."""
        if self.world == 1:
            return
        if self.dist.get_backend() == "nccl":
            if getattr(self, "_fence_t", None) is None:
                self._fence_t = torch.zeros(1, dtype=torch.int32, device=torch.cuda.current_device())
            self.dist.all_reduce(self._fence_t)
            return
        torch.cuda.synchronize()
        self.dist.barrier()

    def close_windows(self):
        pass  # mappings stay cached (see window)

    def account(self, remote: list, rec_bytes: int):
        pass

    def all_to_all_v(self, sends: list, counts: list) -> list:
        send, sc = sends[0], [int(c) for c in counts[0]]
        sct = torch.tensor(sc, dtype=torch.int64, device=send.device)
        rct = torch.empty_like(sct)
        self.dist.all_to_all_single(rct, sct)
        rc = [int(x) for x in rct.tolist()]
        recv = torch.empty((sum(rc),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=rc, input_split_sizes=sc)
        return [recv]


class LocalComm:
    """W ranks emulated in one process (their states are processed in turn)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def all_reduce(self, ts: list, op: str):
        acc = ts[0].clone()
        for t in ts[1:]:
            acc = acc + t if op == "sum" else (torch.maximum(acc, t) if op == "max" else torch.minimum(acc, t))
        for t in ts:
            t.copy_(acc)

    def all_gather(self, ts: list) -> list:
        return [[t.clone() for t in ts] for _ in ts]

    def window(self, ts: list, key: str = "") -> list:
        """Peer window of the emulated ranks: their tensors live on one device."""
        return [list(ts) for _ in ts]

    def fence(self):
        pass  # the emulated ranks' kernels run in order on one stream

    def close_windows(self):
        pass

    def account(self, remote: list, rec_bytes: int):
        pass

    def all_to_all_v(self, sends: list, counts: list) -> list:
        offs = [np.concatenate([[0], np.cumsum([int(c) for c in cs])]).astype(np.int64) for cs in counts]
        return [torch.cat([sends[s][offs[s][d]:offs[s][d + 1]] for s in range(self.world)], 0)
                for d in range(self.world)]


def balanced_splits(hist: np.ndarray, bins: np.ndarray, world: int) -> np.ndarray:
    """Key-range boundaries (node ids, W+1 entries) at histogram-bin edges with
    about equal occurrence counts per rank."""
    cum = np.concatenate([[0], np.cumsum(hist.astype(np.int64))])
    out = [int(bins[0])]
    for r in range(1, world):
        k = int(np.searchsorted(cum, cum[-1] * r / world))
        out.append(max(out[-1], int(bins[min(k, len(bins) - 1)])))
    out.append(int(bins[-1]))
    return np.asarray(out, dtype=np.int32)


# coarse key-range histogram over every HIST_SAMPLE-th element of meshes with
# at least HIST_SAMPLE_MIN_ELEMENTS elements (module constants: tests force it)
HIST_SAMPLE = 8
HIST_SAMPLE_MIN_ELEMENTS = 1 << 20
# halo exchanges of the refined level through peer windows (CUDA backends);
# False: the all-to-all form (tests run both)
P2P = True


def element_splits(nE: int, world: int) -> np.ndarray:
    return np.asarray([nE * r // world for r in range(world + 1)], dtype=np.int32)


# ---- CUDA backend -------------------------------------------------------------------
class CudaRankOps:
    """One rank's operations through the C ABI.  Exchange buffers are torch
    tensors on the rank's device; the ctx must run on torch's current stream
    (dist.py passes it) so kernels and collectives are stream-ordered."""

    def __init__(self, ctx: capi.Context, device):
        self.ctx, self.lib, self.dev = ctx, ctx.lib, torch.device(device)
        self._ee_next = None  # the next level's elem_edge of the own elements

    def _ck(self, st):
        self.ctx.check(st)

    @staticmethod
    def p(t):
        return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None

    def empty(self, shape, dtype=torch.int32):
        return torch.empty(shape, dtype=dtype, device=self.dev)

    def as_tensor(self, a, dtype=torch.int32):
        return torch.as_tensor(np.ascontiguousarray(a)).to(device=self.dev, dtype=dtype)

    def mesh_view(self, coords, nC, elements, nE_local, nE_cols):
        """phfem_mesh over replicated coordinates and the rank's elements;
        nE_cols = global element count (columns of C are 3 m, m global)."""
        m = capi.phfem_mesh()
        m.coords, m.elements = coords.data_ptr(), (elements.data_ptr() if elements.numel() else None)
        m.nC, m.nE, m.nD, m.nN = nC, nE_local, 0, 0
        m.owned = 0
        self._cols = nE_cols
        return m

    # -- edge dedup -------------------------------------------------------------------
    def occurrences(self, elements, elo, ehi, splits, pack: bool):
        W = splits.numel() - 1
        cnt = self.empty(W)
        if not pack:
            self._ck(self.lib.phfem_dist_occurrences(self.ctx.ptr, self.p(elements), elo, ehi, self.p(splits), W,
                                                     self.p(cnt), None, None))
            return cnt
        off = self.empty(W + 1)
        send = self.empty((max(3 * (ehi - elo), 1), 4))
        self._ck(self.lib.phfem_dist_occurrences(self.ctx.ptr, self.p(elements), elo, ehi, self.p(splits), W,
                                                 self.p(cnt), self.p(off), self.p(send)))
        return send[:3 * (ehi - elo)], cnt.tolist()

    # -- input level through peer windows (phfem_dist_bucket_* / scatter_p2p) ------
    def bucket_bits(self, nC, nE):
        return int(self.lib.phfem_dist_bucket_bits(nC, nE))

    def bucket_hist(self, elements, elo, nC, nE, NB):
        hist = self.empty((NB,))
        self._ck(self.lib.phfem_dist_bucket_hist(self.ctx.ptr, self.p(elements), int(elements.shape[0]), elo, nC, nE,
                                                 self.p(hist)))
        return hist

    def bucket_cursors(self, hist_all, me, bsplits):
        W, NB = int(hist_all.shape[0]), int(hist_all.shape[1])
        b = bsplits.cpu().tolist()
        self._cursor = self.empty((NB,))
        self._boff = self.empty((b[me + 1] - b[me] + 1,))
        n = C.c_int64(0)
        self._ck(self.lib.phfem_dist_bucket_cursors(self.ctx.ptr, self.p(hist_all.contiguous()), W, NB, me,
                                                    self.p(bsplits), self.p(self._cursor), self.p(self._boff),
                                                    C.byref(n)))
        return int(n.value)

    def items_alloc(self, n):
        self._items = self._buffer("_items_buf", n, dtype=torch.int64)
        return self._items

    def scatter_p2p(self, elements, elo, nC, nE, bsplits, peers, me):
        W = len(peers)
        ptrs, remote = self._ptrs(peers), self.empty(W)
        self._ck(self.lib.phfem_dist_scatter_p2p(self.ctx.ptr, self.p(elements), int(elements.shape[0]), elo, nC, nE,
                                                 self.p(self._cursor), self.p(bsplits), W, me, self.p(ptrs),
                                                 self.p(remote)))
        self._keep = ptrs
        return remote

    def dedup_items(self, n, nlo, nhi, nC, nE, own_range):
        """the owner's tile / emit passes over the items the ranks stored into
        its window (own elements' elem_edge in place, the others as pairs)"""
        pairs = self.empty((max(2 * n, 1), 2))
        t = capi.phfem_topology()
        npairs = C.c_int64(0)
        lo, hi = own_range
        ee = self._buffer("_ee_buf", hi - lo, (3,))  # persistent: the element owner's peer window
        self._ck(self.lib.phfem_dist_dedup_items(self.ctx.ptr, self.p(self._items), n, self.p(self._boff), nlo, nhi,
                                                 nC, nE, lo, hi, self.p(ee), C.byref(t), self.p(pairs),
                                                 C.byref(npairs)))
        self._cursor = self._boff = None
        self.part = capi.Topology(self.ctx, t)
        self.pairs = pairs[:int(npairs.value)]
        self._pairs = (pairs.data_ptr(), int(npairs.value), False)
        self._ee_next = ee[:hi - lo]
        return int(t.E), int(t.n_boundary)

    def dedup(self, recv, nlo, nhi, nC, nE, own_range=None):
        """own_range = the rank's elements [lo, hi): their elem_edge entries are
        written in place (local ids, re-based in route_pairs); only the other
        ranks' entries leave as pairs."""
        n = recv.shape[0]
        pairs = self.empty((max(2 * n, 1), 2))
        t = capi.phfem_topology()
        npairs = C.c_int64(0)
        lo, hi = own_range if own_range is not None else (0, 0)
        ee = self.empty((max(hi - lo, 1), 3)) if own_range is not None else None
        self._ck(self.lib.phfem_dist_dedup_ex(self.ctx.ptr, self.p(recv), n, nlo, nhi, nC, nE, lo, hi,
                                              self.p(ee) if ee is not None else None, C.byref(t), self.p(pairs),
                                              C.byref(npairs)))
        self.part = capi.Topology(self.ctx, t)
        self.pairs = pairs[:int(npairs.value)]
        self._pairs = (pairs.data_ptr(), int(npairs.value), False)
        self._ee_next = ee[:hi - lo] if ee is not None else None
        return int(t.E), int(t.n_boundary)

    # -- refined level, halo form (phfem_dist_side_* / _start_* / _children_slots) ----
    def side_records(self, elements, elem_edge, esplits):
        """element owner: one 16-byte side record per element slot, routed to
        the owner of the slot's parent edge"""
        n = int(elements.shape[0])
        W = esplits.numel() - 1
        cnt, off = self.empty(W), self.empty(W + 1)
        send = self.empty((max(3 * n, 1), 4))
        self._ck(self.lib.phfem_dist_side_records(self.ctx.ptr, self.p(elements), self.p(elem_edge), n,
                                                  self.p(esplits), W, self.p(cnt), self.p(off), self.p(send)))
        return send[:3 * n], cnt.tolist()

    def side_apply(self, recv, E0):
        E = int(self.part.t.E)
        self._side = self.empty((max(2 * E, 1), 4))   # t_minus entries of boundary edges stay unused
        self._ck(self.lib.phfem_dist_side_apply(self.ctx.ptr, self.p(recv), int(recv.shape[0]), E0, E,
                                                self.p(self._side)))

    def refine_level_side(self, coords, nc, E0p, nlo, nhi, nE_all, coords_fine, neu_parent=None):
        """edge owner: the fine part of its parent edges (local ids), their rank
        bytes, owned midpoints into coords_fine; C's rows when neu_parent is
        given (the last level).  The parent part is kept for start_records."""
        pt = self.part.t
        E = int(pt.E)
        rk = torch.empty((max(E, 1),), dtype=torch.uint8, device=self.dev)
        t = capi.phfem_topology()
        csr = capi.phfem_csr() if neu_parent is not None else None
        nN = 0 if neu_parent is None else int(neu_parent.numel())
        self._ck(self.lib.phfem_dist_refine_level_side(
            self.ctx.ptr, C.byref(pt), E0p, self.p(self._side), self.p(coords), nc, nlo, nhi, nE_all,
            self.p(neu_parent) if nN else None, nN, C.byref(t), self.p(rk), self.p(coords_fine),
            C.byref(csr) if csr is not None else None))
        if csr is not None:
            self.csr = csr
        self._side = None
        self.ppart, self.part, self._rk = self.part, capi.Topology(self.ctx, t), rk
        return int(t.E), int(t.n_boundary)

    def level_count(self, E0p, neu_parent=None):
        """count half of the level: (fine edges, parent Neumann edges) of the rank"""
        Ef, nneu, plan = C.c_int32(0), C.c_int32(0), C.c_void_p()
        nN = 0 if neu_parent is None else int(neu_parent.numel())
        self._ck(self.lib.phfem_dist_level_count(self.ctx.ptr, C.byref(self.part.t), E0p, self.p(self._side),
                                                 self.p(neu_parent) if nN else None, nN,
                                                 1 if neu_parent is not None else 0, C.byref(Ef), C.byref(nneu),
                                                 C.byref(plan)))
        self._plan, self._plan_C = plan, neu_parent is not None
        return int(Ef.value), int(nneu.value)

    def level_run(self, coords, nc, nlo, nhi, nE_all, coords_fine, f_off, nnz_off):
        """run half: the fine part with GLOBAL ids (f_off, nnz_off) — no re-basing"""
        E = int(self.part.t.E)
        rk = torch.empty((max(E, 1),), dtype=torch.uint8, device=self.dev)
        t = capi.phfem_topology()
        csr = capi.phfem_csr() if self._plan_C else None
        plan, self._plan = self._plan, None
        self._ck(self.lib.phfem_dist_level_run(self.ctx.ptr, plan, self.p(coords), nc, nlo, nhi, nE_all, f_off,
                                               nnz_off, C.byref(t), self.p(rk), self.p(coords_fine),
                                               C.byref(csr) if csr is not None else None))
        if csr is not None:
            self.csr = csr
        self._side = None
        self.ppart, self.part, self._rk = self.part, capi.Topology(self.ctx, t), rk
        return int(t.E), int(t.n_boundary)

    def start_records(self, nes_off, psplits):
        """edge owner: {slot, group start (global), rank byte} per (owned parent
        edge, element), routed to the element owners; drops the parent part"""
        pt = self.ppart.t
        W = psplits.numel() - 1
        cnt, off = self.empty(W), self.empty(W + 1)
        send = self.empty((max(2 * int(pt.E), 1), 3))
        self._ck(self.lib.phfem_dist_start_records(self.ctx.ptr, C.byref(pt),
                                                   C.c_void_p(self.part.t.node_edge_start), nes_off,
                                                   self.p(self._rk), self.p(psplits), W, self.p(cnt),
                                                   self.p(off), self.p(send)))
        self.ppart.release()
        self.ppart, self._rk = None, None
        c = cnt.tolist()
        return send[:sum(c)], c

    def start_apply(self, recv, elo, n):
        gs = self.empty((max(3 * n, 1),))
        grk = torch.empty((max(3 * n, 1),), dtype=torch.uint8, device=self.dev)
        self._ck(self.lib.phfem_dist_start_apply(self.ctx.ptr, self.p(recv), int(recv.shape[0]), elo, self.p(gs),
                                                 self.p(grk)))
        return gs, grk

    def children_slots(self, elements, elem_edge, gs, grk, nc, coords_fine, own=(0, 0)):
        """own: the rank's parent edge range (their midpoints: its level kernel's)"""
        n = int(elements.shape[0])
        kids = self.empty((max(4 * n, 1), 3))
        ee = self.empty((max(4 * n, 1), 3))
        self._ck(self.lib.phfem_dist_children_slots_ex(self.ctx.ptr, self.p(elements), self.p(elem_edge), n,
                                                       self.p(gs), self.p(grk), nc, int(own[0]), int(own[1]), None,
                                                       0, None, self.p(coords_fine), self.p(kids), self.p(ee)))
        return kids[:4 * n], ee[:4 * n]

    # -- peer-window forms (phfem_dist_side_p2p / _start_p2p) ---------------------------
    def _ptrs(self, ts):
        return torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=self.dev)

    def _buffer(self, name, n, shape_tail=(), dtype=torch.int32):
        """persistent exchange buffer (the peer windows map it once)"""
        b = getattr(self, name, None)
        if b is None or b.shape[0] < n:
            b = torch.empty((max(n, 1),) + shape_tail, dtype=dtype, device=self.dev)
            setattr(self, name, b)
        return b[:max(n, 1)]

    def side_alloc(self):
        self._side = self._buffer("_side_buf", 2 * int(self.part.t.E), (4,))
        return self._side

    def side_p2p(self, elements, elem_edge, esplits, peers, me):
        """side records stored straight into the edge owners' side arrays"""
        n, W = int(elements.shape[0]), len(peers)
        ptrs, remote = self._ptrs(peers), self.empty(W)
        self._ck(self.lib.phfem_dist_side_p2p(self.ctx.ptr, self.p(elements), self.p(elem_edge), n, self.p(esplits),
                                              W, me, self.p(ptrs), self.p(remote)))
        self._keep = ptrs
        return remote

    def start_alloc(self, n):
        self._gs = self._buffer("_gs_buf", 3 * n)
        self._grk = self._buffer("_grk_buf", 3 * n, dtype=torch.uint8)
        return self._gs, self._grk

    def start_p2p(self, nes_off, psplits, peers_gs, peers_grk, me):
        """group-start records stored straight into the element owners' slots"""
        pt = self.ppart.t
        W = len(peers_gs)
        pg, pr, remote = self._ptrs(peers_gs), self._ptrs(peers_grk), self.empty(W)
        self._ck(self.lib.phfem_dist_start_p2p(self.ctx.ptr, C.byref(pt), C.c_void_p(self.part.t.node_edge_start),
                                               nes_off, self.p(self._rk), self.p(psplits), W, me, self.p(pg),
                                               self.p(pr), self.p(remote)))
        self._keep = (pg, pr)
        self.ppart.release()
        self.ppart, self._rk = None, None
        return remote

    def route_pairs(self, E0, esplits, elo, ehi):
        """Pairs of the own (destination-level) elements [elo, ehi) go straight
        into the next elem_edge; the rest is packed by owner for the exchange."""
        W = esplits.numel() - 1
        ptr, n, owned = self._pairs
        cnt, off = self.empty(W), self.empty(W + 1)
        send = self.empty((max(n, 1), 2))
        if self._ee_next is None:
            self._ee_next = self.empty((ehi - elo, 3))
        elif E0 and ehi > elo:  # written in place by the level kernel with local ids
            self.rebase(self._ee_next.data_ptr(), 3 * (ehi - elo), E0, 2)
        self._ck(self.lib.phfem_dist_route_pairs(self.ctx.ptr, C.c_void_p(ptr) if n else None, n, E0,
                                                 self.p(esplits), W, self.p(cnt), self.p(off), self.p(send), elo, ehi,
                                                 self.p(self._ee_next)))
        if owned:
            self.ctx.free(ptr)
        self._pairs = (0, 0, False)
        self.pairs = None
        c = cnt.tolist()
        return send[:sum(c)], c

    def ee_window(self):
        return self._ee_next

    def rebase_own_ee(self, E0, elo, ehi):
        """own entries (local ids from the emit pass) -> global; must precede
        the peers' stores into this window (they store global ids)"""
        if E0 and ehi > elo:
            self.rebase(self._ee_next.data_ptr(), 3 * (ehi - elo), E0, 2)

    def pairs_p2p(self, E0, esplits, peers, me):
        """the other ranks' entries stored straight into their elem_edge windows"""
        ptr, n, owned = self._pairs
        W = len(peers)
        pp, remote = self._ptrs(peers), self.empty(W)
        self._ck(self.lib.phfem_dist_pairs_p2p(self.ctx.ptr, C.c_void_p(ptr) if n else None, n, E0, self.p(esplits),
                                               W, me, self.p(pp), self.p(remote)))
        if owned:
            self.ctx.free(ptr)
        self._pairs = (0, 0, False)
        self.pairs = None
        self._keep = pp
        return remote

    def take_ee(self):
        ee, self._ee_next = self._ee_next, None
        return ee

    def apply_pairs(self, recv, elo, ehi):
        ee, self._ee_next = self._ee_next, None
        self._ck(self.lib.phfem_dist_apply_pairs(self.ctx.ptr, self.p(recv), recv.shape[0], elo, self.p(ee)))
        return ee

    def rebase(self, ptr, n, off, only_nonneg=0):
        self._ck(self.lib.phfem_dist_add_offset(self.ctx.ptr, C.c_void_p(ptr), n, off, only_nonneg))

    def rebase_part(self, E0):
        t = self.part.t
        for ptr, n in ((t.interior_edges, t.n_interior), (t.boundary_edges, t.n_boundary),
                       (t.node_edge_start, t.nC + 1)):
            if n:
                self.rebase(ptr, n, E0)

    def resolve(self, pairs, list_base, nlo, E0):
        n = pairs.shape[0]
        ids = torch.full((max(n, 1),), -1, dtype=torch.int32, device=self.dev)
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        if n:
            self._ck(self.lib.phfem_dist_resolve(self.ctx.ptr, C.byref(self.part.t), nlo, E0, self.p(pairs), n,
                                                 list_base, self.p(ids), self.p(err)))
        return ids[:n], err

    # -- refinement -----------------------------------------------------------------
    def midpoints(self, coords):
        t = self.part.t
        out = self.empty((max(t.E, 1), 2), torch.float64)
        self._ck(self.lib.phfem_dist_midpoints(self.ctx.ptr, self.p(coords), C.c_void_p(t.edge_nodes), t.E,
                                               self.p(out)))
        return out[:t.E]

    def children(self, elements, elem_edge, nC):
        n = elements.shape[0]
        out = self.empty((max(4 * n, 1), 3))
        self._ck(self.lib.phfem_dist_children(self.ctx.ptr, self.p(elements), self.p(elem_edge), n, nC,
                                              self.p(out)))
        return out[:4 * n]

    # -- classification, C, boundary vectors, blocks ------------------------------------------
    def classify(self, dir_ids_local, neu_ids_local, E0, R0=None):
        """R0 given (offsets known before): retained positions / edges global at once"""
        c = capi.phfem_classification()
        self._ck(self.lib.phfem_dist_classify_ex(self.ctx.ptr, C.byref(self.part.t), E0, self.p(dir_ids_local),
                                                 dir_ids_local.numel(), self.p(neu_ids_local), neu_ids_local.numel(),
                                                 0 if R0 is None else R0, 0 if R0 is None else E0, C.byref(c)))
        self.cls = capi.Classification(self.ctx, c)
        self._r_off = R0 or 0
        return int(c.L)

    def constraint(self, mview):
        if getattr(self, "csr", None) is not None:  # fused into the refined level
            return self.csr
        m = capi.phfem_csr()
        mv = capi.phfem_mesh()
        C.memmove(C.byref(mv), C.byref(mview), C.sizeof(mv))
        mv.nE = self._cols
        self._ck(self.lib.phfem_assemble_constraint(self.ctx.ptr, C.byref(mv), C.byref(self.part.t),
                                                    C.byref(self.cls.c), C.byref(m)))
        self.csr = m
        return m

    def dirichlet(self, mview, uD, t):
        bd = self.empty((max(self.cls.c.L, 1),), torch.float64)
        # retained positions global when the classification got R0
        self._ck(self.lib.phfem_dist_dirichlet(self.ctx.ptr, C.byref(mview), C.byref(self.part.t),
                                               C.byref(self.cls.c), C.byref(uD), t, getattr(self, "_r_off", 0),
                                               self.p(bd)))
        return bd[:self.cls.c.L]

    def volume(self, mview, coeffs, f, t):
        n = mview.nE
        out = {k: self.empty((max(n, 1), 9), torch.float64) for k in ("B", "D", "M", "M0")}
        load = self.empty((max(n, 1), 3), torch.float64)
        self._ck(self.lib.phfem_assemble_volume_load(self.ctx.ptr, C.byref(mview), C.byref(coeffs), C.byref(f), t,
                                                     self.p(out["B"]), self.p(out["D"]), self.p(out["M"]),
                                                     self.p(out["M0"]), self.p(load)))
        out = {k: v[:n] for k, v in out.items()}
        out["load"] = load[:n]
        return out

    def volume_start(self, mview, coeffs, f, t):
        """the blocks + load of the own elements on a side stream, so they
        overlap the host-synchronised classification / resolve / Neumann phases
        of the last level (they need only the own elements and coordinates)"""
        main = torch.cuda.current_stream(self.dev)
        if getattr(self, "_side_stream", None) is None:
            self._side_stream = torch.cuda.Stream(device=self.dev)
            self._side_ctx = capi.Context(self.ctx.device, stream=self._side_stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(main)
        self._side_stream.wait_event(ev)
        n = mview.nE
        out = {k: self.empty((max(n, 1), 9), torch.float64) for k in ("B", "D", "M", "M0")}
        load = self.empty((max(n, 1), 3), torch.float64)
        for x in list(out.values()) + [load]:
            x.record_stream(self._side_stream)
        self._side_keep = (mview, self.p(out["B"]))
        self._side_ctx.check(self.lib.phfem_assemble_volume_load(
            self._side_ctx.ptr, C.byref(mview), C.byref(coeffs), C.byref(f), t, self.p(out["B"]), self.p(out["D"]),
            self.p(out["M"]), self.p(out["M0"]), self.p(load)))
        self._vol_done = torch.cuda.Event()
        self._vol_done.record(self._side_stream)
        out = {k: v[:n] for k, v in out.items()}
        out["load"] = load[:n]
        return out

    def volume_join(self):
        if getattr(self, "_vol_done", None) is not None:
            torch.cuda.current_stream(self.dev).wait_event(self._vol_done)
            self._vol_done = None

    def neumann_table(self, neu_ids_local, nN_all, positions):
        """rows {a, b, t_plus, led} of the owned Neumann edges at their global
        list positions (others zero)."""
        table = torch.zeros((max(nN_all, 1), 4), dtype=torch.int32, device=self.dev)
        if nN_all:
            full = torch.full((nN_all,), -1, dtype=torch.int32, device=self.dev)
            full[positions] = neu_ids_local
            self._ck(self.lib.phfem_dist_neumann_table(self.ctx.ptr, C.byref(self.part.t), 0, self.p(full), nN_all,
                                                       self.p(table)))
        return table[:nN_all]

    def neumann_apply(self, mview, table, dup, elo, ehi, g, t, load):
        self._ck(self.lib.phfem_dist_neumann_apply(self.ctx.ptr, C.byref(mview), self.p(table), table.shape[0],
                                                   1 if dup else 0, elo, ehi, C.byref(g), t, self.p(load)))

    def num_edges(self) -> int:
        return int(self.part.t.E)

    def rebase_results(self, E0, R0, nnz0, retained=True, row_ptr=True):
        """rank-local retained positions / retained edges / CSR row pointers -> global
        (skipped for what the level / classification already wrote globally)"""
        c, m = self.cls.c, self.csr
        if retained and c.E:
            self.rebase(c.retained_pos, c.E, R0, 1)
        if retained and c.L:
            self.rebase(c.retained_edges, c.L, E0)
        if row_ptr:
            self.rebase(m.row_ptr, m.rows + 1, nnz0)

    # -- results -----------------------------------------------------------------------------------
    def part_arrays(self) -> dict:
        d = self.part.download()
        d.pop("elem_edge", None)
        return d

    def cls_arrays(self) -> dict:
        return self.cls.download()

    def csr_arrays(self):
        m, x = self.csr, self.ctx
        return (x.to_host(m.row_ptr, (m.rows + 1,), np.int32), x.to_host(m.col_idx, (m.nnz,), np.int32),
                x.to_host(m.values, (m.nnz,), np.float64))

    def release(self):
        if getattr(self, "csr", None) is not None:
            self.lib.phfem_csr_release(self.ctx.ptr, C.byref(self.csr))
            self.csr = None
        for a in ("cls", "part"):
            o = getattr(self, a, None)
            if o is not None:
                o.release()
                setattr(self, a, None)


# ---- one rank's state -------------------------------------------------------------------
@dataclass
class RankState:
    rank: int
    ops: object
    coords: torch.Tensor        # replicated [nC][2] fp64
    elements: torch.Tensor      # own elements [n][3] int32
    elo: int
    ehi: int
    dirichlet: torch.Tensor     # replicated boundary lists [nD][2], [nN][2]
    neumann: torch.Tensor


def _edge_generation(states: List[RankState], comm, nC: int, nE: int, esplits: np.ndarray,
                     nbins_per_rank: int = 64):
    """Distributed build_topology.  Returns the key-range splits, per-state
    (E0, B0) and the global (E, n_boundary); each ops holds its part (global
    ids) and each state gets its elem_edge."""
    W = comm.world
    tr = getattr(comm, "trace", None) or (lambda w: None)
    nb = max(1, min(nbins_per_rank * W, 4096, nC))  # key ranges balanced to ~1/64 of a share
    bins = np.asarray([nC * i // nb for i in range(nb + 1)], dtype=np.int32)
    # coarse histogram of max nodes -> balanced key ranges (identical on every rank)
    # the key ranges only balance the work (no output depends on them): a
    # 1/8 sample of the own elements is enough for the coarse histogram
    S = HIST_SAMPLE if nE >= HIST_SAMPLE_MIN_ELEMENTS else 1
    smp = [s.elements[::S].contiguous() if S > 1 else s.elements for s in states]
    hists = [s.ops.occurrences(e, 0, int(e.shape[0]), s.ops.as_tensor(bins), pack=False)
             for s, e in zip(states, smp)]
    comm.all_reduce(hists, "sum")
    splits = balanced_splits(hists[0].cpu().numpy(), bins, W)
    tr("hist")
    eb = []
    p2p = P2P and hasattr(states[0].ops, "scatter_p2p")
    if p2p:
        # key ranges on 256-node tile boundaries: every MSD bucket has one owner
        # and its global index is max >> bs; the ranks store their packed
        # occurrences straight into the owners' bucket arrays (peer windows)
        splits = np.asarray([0] + [int(x) // 256 * 256 for x in splits[1:-1]] + [nC], dtype=np.int32)
        bs = states[0].ops.bucket_bits(nC, nE)
        NB = (nC + (1 << bs) - 1) >> bs
        bsplits = np.asarray([int(x) >> bs for x in splits[:-1]] + [NB], dtype=np.int32)
        hists = [s.ops.bucket_hist(s.elements, s.elo, nC, nE, NB) for s in states]
        gh = comm.all_gather(hists)
        nitems = [s.ops.bucket_cursors(torch.stack(g), s.rank, s.ops.as_tensor(bsplits)) for s, g in zip(states, gh)]
        wins = comm.window([s.ops.items_alloc(n) for s, n in zip(states, nitems)], "items")
        rem = [s.ops.scatter_p2p(s.elements, s.elo, nC, nE, s.ops.as_tensor(bsplits), w, s.rank)
               for s, w in zip(states, wins)]
        comm.fence()
        comm.account(rem, 8)
        tr("scatter")
        for s, n in zip(states, nitems):
            r = s.rank
            E_r, B_r = s.ops.dedup_items(n, int(splits[r]), int(splits[r + 1]), nC, nE, own_range=(s.elo, s.ehi))
            eb.append(torch.tensor([E_r, B_r], dtype=torch.int64, device=s.coords.device))
        tr("dedup")
    else:
        # forward all-to-all of the occurrences, local dedup
        packed = [s.ops.occurrences(s.elements, s.elo, s.ehi, s.ops.as_tensor(splits), pack=True) for s in states]
        tr("pack")
        recvs = comm.all_to_all_v([p[0] for p in packed], [p[1] for p in packed])
        tr("a2a")
        for s, rv in zip(states, recvs):
            r = s.rank
            E_r, B_r = s.ops.dedup(rv, int(splits[r]), int(splits[r + 1]), nC, nE, own_range=(s.elo, s.ehi))
            eb.append(torch.tensor([E_r, B_r], dtype=torch.int64, device=s.coords.device))
        tr("dedup")
    gath = comm.all_gather(eb)
    per = []
    for s, g in zip(states, gath):
        allc = torch.stack(g).cpu().numpy()
        E0, B0 = int(allc[:s.rank, 0].sum()), int(allc[:s.rank, 1].sum())
        per.append((E0, B0))
        s.ops.rebase_part(E0)
    Etot, Btot = int(allc[:, 0].sum()), int(allc[:, 1].sum())
    if p2p:
        # (slot, global edge id) stored straight into the element owners' elem_edge
        wins = comm.window([s.ops.ee_window() for s in states], "ee")
        for s, (E0, _) in zip(states, per):
            s.ops.rebase_own_ee(E0, s.elo, s.ehi)
        comm.fence()   # every rank's own entries final before the peers store theirs
        rem = [s.ops.pairs_p2p(E0, s.ops.as_tensor(esplits), w, s.rank)
               for s, (E0, _), w in zip(states, per, wins)]
        comm.fence()
        comm.account(rem, 4)
        for s in states:
            s.elem_edge = s.ops.take_ee()
        tr("pairs")
    else:
        # reverse all-to-all: (element slot, global edge id) to the element owners
        routed = [s.ops.route_pairs(E0, s.ops.as_tensor(esplits), s.elo, s.ehi) for s, (E0, _) in zip(states, per)]
        recvs = comm.all_to_all_v([x[0] for x in routed], [x[1] for x in routed])
        tr("route")
        for s, rv in zip(states, recvs):
            s.elem_edge = s.ops.apply_pairs(rv, s.elo, s.ehi)
        tr("pairs")
    return splits, per, (Etot, Btot)


def _resolve(states, comm, splits, per, nD, nN):
    """Global boundary-pair ids (every rank) + the reference's first error."""
    ids = []
    errs = []
    for s, (E0, _) in zip(states, per):
        pairs = torch.cat([s.dirichlet, s.neumann], 0).reshape(-1, 2).contiguous()
        i, e = s.ops.resolve(pairs, 0, int(splits[s.rank]), E0)
        ids.append(i.to(torch.int64))
        errs.append(e)
    if nD + nN:
        comm.all_reduce(ids, "max")
        # ~0 (no error) is -1 as int64: shift to make "no error" the largest
        shifted = [torch.where(e == -1, torch.full_like(e, 2 ** 62), e) for e in errs]
        comm.all_reduce(shifted, "min")
        key = int(shifted[0].item())
        if key != 2 ** 62:
            pos, interior = key >> 2, key & 1
            s = states[0]
            is_d = pos < nD
            pr = (s.dirichlet[pos] if is_d else s.neumann[pos - nD]).tolist()
            what = "dirichlet" if is_d else "neumann"
            raise RuntimeError(f"{what} pair ({pr[0] + 1},{pr[1] + 1}) " +
                               ("resolves to an interior edge" if interior else "is not an edge"))
    return ids


def _gather_rows(comm, ts: list) -> list:
    """All-gather of per-rank row blocks of different lengths -> the full
    array (rank order) on every rank."""
    if comm.world == 1:
        return [t.contiguous() for t in ts]
    counts = [torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device) for t in ts]
    cg = comm.all_gather(counts)
    nmax = max(1, max(int(torch.stack(c).max().item()) for c in cg))
    padded = [torch.cat([t, t.new_zeros((nmax - t.shape[0],) + tuple(t.shape[1:]))], 0) for t in ts]
    gm = comm.all_gather(padded)
    return [torch.cat([p[:int(n.item())] for p, n in zip(parts, c)], 0).contiguous() for parts, c in zip(gm, cg)]


def _bisect(pairs, eid, nC):
    """refine.cpp:39-50: boundary pair (a, b) of edge e -> (a, mid), (mid, b)"""
    if pairs.shape[0] == 0:
        return pairs
    mid = (eid + nC).to(pairs.dtype)
    return torch.stack([pairs[:, 0], mid, mid, pairs[:, 1]], 1).reshape(-1, 2).contiguous()


def _refine_sorted(states, comm, nC, splits, per, Etot, nD, nN, ids):
    """One refinement with the refined topology left to the next (sort-based)
    edge generation: midpoints of the owned edges, all-gathered."""
    mids = _gather_rows(comm, [s.ops.midpoints(s.coords) for s in states])
    for s, m, i in zip(states, mids, ids):
        kids = s.ops.children(s.elements, s.elem_edge, nC)
        s.dirichlet, s.neumann = _bisect(s.dirichlet, i[:nD], nC), _bisect(s.neumann, i[nD:], nC)
        s.ops.release()
        s.coords, s.elements = torch.cat([s.coords, m], 0).contiguous(), kids
        s.elo, s.ehi = 4 * s.elo, 4 * s.ehi


def _refine_sort_free(states, comm, nC, nE, splits, per, Etot, Btot, esplits, nD, nN, ids, fused_c=False,
                      last=False):
    """One refinement with the fine topology straight from the parent's
    (SURVEY f1), halo form — no all-gather of parent arrays or midpoints:
      1. every element owner sends one 16-byte side record per element slot
         {edge, partner edges, opposite vertex} to the owner of the slot's
         parent edge (all-to-all);
      2. edge owners build the groups of their parent edges (fine node range
         [nC + E0, nC + E0 + E_r); rank 0 also holds the old nodes) and write
         their midpoints into their fine coordinate array;
      3. edge owners send {slot, group start, rank byte} per (edge, element)
         back to the element owners (all-to-all, after the fine counts are
         all-gathered);
      4. element owners write the children rows, the fine elem_edge and the
         midpoints of their own elements' edges (same bits) locally.
    Coordinates stay replicated only while another level follows (the owned
    midpoints are all-gathered then); after the last level every rank holds
    the coordinates its elements and edges reference.  Returns the fine
    (splits, per, totals)."""
    tr = getattr(comm, "trace", None) or (lambda w: None)
    E0s = _all_E0(states, comm, per)
    edge_splits = np.asarray(E0s + [Etot], dtype=np.int32)
    # peer windows when the backend has them (CUDA ranks): one kernel per
    # exchange stores every record into its final slot on the owner
    p2p = P2P and hasattr(states[0].ops, "side_p2p")
    if p2p:
        wins = comm.window([s.ops.side_alloc() for s in states], "side")
        rem = [s.ops.side_p2p(s.elements, s.elem_edge, s.ops.as_tensor(edge_splits), w, s.rank)
               for s, w in zip(states, wins)]
        comm.fence()
        comm.account(rem, 16)
    else:
        sides = [s.ops.side_records(s.elements, s.elem_edge, s.ops.as_tensor(edge_splits)) for s in states]
        recvs = comm.all_to_all_v([x[0] for x in sides], [x[1] for x in sides])
        for s, rv, (E0, _) in zip(states, recvs, per):
            s.ops.side_apply(rv, E0)
    tr("side")
    # fine node ranges from every rank's parent edge offset
    fsplits = np.asarray([0] + [nC + e for e in E0s[1:]] + [nC + Etot], dtype=np.int64)
    for s in states:
        cf = torch.empty((nC + Etot, 2), dtype=torch.float64, device=s.coords.device)
        cf[:nC] = s.coords[:nC]
        s.coords_fine = cf
    neus = [i[nD:].to(torch.int32).contiguous() if fused_c else None for i in ids]
    fper = []
    if hasattr(states[0].ops, "level_count"):
        # count half first: every rank's fine offsets (edges, C rows / entries)
        # are all-gathered before the level kernel writes, so it writes global
        # ids — no re-basing pass over the fine part or C's row pointers
        counts = []
        for s, (E0, _), neu in zip(states, per, neus):
            Ef_r, nneu_r = s.ops.level_count(E0, neu)
            Bf_r = 2 * int(s.ops.part.t.n_boundary)
            counts.append(torch.tensor([Ef_r, Bf_r, nneu_r], dtype=torch.int64, device=s.coords.device))
        gath = comm.all_gather(counts)
        for s, gc in zip(states, gath):
            allc = torch.stack(gc).cpu().numpy()
            r = s.rank
            E0f, B0f = int(allc[:r, 0].sum()), int(allc[:r, 1].sum())
            N0f = 2 * int(allc[:r, 2].sum())            # fine Neumann edges before the rank
            R0 = E0f - N0f                              # retained rows before it
            nnz0 = 4 * R0 - 2 * (B0f - N0f) if fused_c else 0
            fper.append((E0f, B0f))
            s.ops.level_run(s.coords, nC, int(fsplits[r]), int(fsplits[r + 1]), nE, s.coords_fine, E0f, nnz0)
            s.fine_offsets = (E0f, R0) if fused_c else None
        Ef_tot, Bf_tot = int(allc[:, 0].sum()), int(allc[:, 1].sum())
    else:
        counts = []
        for s, (E0, _), neu in zip(states, per, neus):
            r = s.rank
            Ef, Bf = s.ops.refine_level_side(s.coords, nC, E0, int(fsplits[r]), int(fsplits[r + 1]), nE,
                                             s.coords_fine, neu)
            counts.append(torch.tensor([Ef, Bf], dtype=torch.int64, device=s.coords.device))
        gath = comm.all_gather(counts)
        for s, gc in zip(states, gath):
            allc = torch.stack(gc).cpu().numpy()
            E0f, B0f = int(allc[:s.rank, 0].sum()), int(allc[:s.rank, 1].sum())
            fper.append((E0f, B0f))
            s.ops.rebase_part(E0f)
        Ef_tot, Bf_tot = int(allc[:, 0].sum()), int(allc[:, 1].sum())
    tr("level")
    if p2p:
        bufs = [s.ops.start_alloc(s.ehi - s.elo) for s in states]
        wg, wr = comm.window([b[0] for b in bufs], "gs"), comm.window([b[1] for b in bufs], "grk")
        rem = [s.ops.start_p2p(nC + E0 - int(fsplits[s.rank]), s.ops.as_tensor(esplits), g_, r_, s.rank)
               for s, (E0, _), g_, r_ in zip(states, per, wg, wr)]
        comm.fence()
        comm.account(rem, 5)
    else:
        starts = [s.ops.start_records(nC + E0 - int(fsplits[s.rank]), s.ops.as_tensor(esplits))
                  for s, (E0, _) in zip(states, per)]
        recvs = comm.all_to_all_v([x[0] for x in starts], [x[1] for x in starts])
        bufs = [s.ops.start_apply(rv, s.elo, s.ehi - s.elo) for s, rv in zip(states, recvs)]
    comm.close_windows()
    tr("start")
    for s, (gs, grk), i in zip(states, bufs, ids):
        kids, ee = s.ops.children_slots(s.elements, s.elem_edge, gs, grk, nC, s.coords_fine,
                                        own=(int(edge_splits[s.rank]), int(edge_splits[s.rank + 1])))
        s.dirichlet, s.neumann = _bisect(s.dirichlet, i[:nD], nC), _bisect(s.neumann, i[nD:], nC)
        s.elements, s.elem_edge = kids, ee
        s.elo, s.ehi = 4 * s.elo, 4 * s.ehi
    own = [s.coords_fine[nC + int(edge_splits[s.rank]):nC + int(edge_splits[s.rank + 1])] for s in states]
    if last:
        for s, m in zip(states, own):
            s.nc_parent, s.mid_own = nC, m
            s.coords = s.coords_fine
    else:
        gm = _gather_rows(comm, [m.contiguous() for m in own])
        for s, m in zip(states, gm):
            s.coords = torch.cat([s.coords[:nC], m], 0).contiguous()
    for s in states:
        s.coords_fine = None
    tr("refine")
    return fsplits.astype(np.int32), fper, (Ef_tot, Bf_tot)


def _all_E0(states, comm, per) -> list:
    """E0 of every rank (each rank knows only its own from `per`)."""
    ts = [torch.tensor([E0], dtype=torch.int64, device=s.coords.device) for s, (E0, _) in zip(states, per)]
    g = comm.all_gather(ts)[0]
    return [int(x) for x in torch.cat(g).cpu().tolist()]


def distributed_pipeline(states: List[RankState], comm, nC: int, nE: int, levels: int, coeffs, f, g, uD,
                         t: float = 0.0, sort_free: bool = True):
    """edge generation -> [red refinement + refined topology] x levels ->
    classification -> B, D, M, M0, load = b + LN, C (CSR rows), bD; every rank
    keeps its slices (collect() gathers them for tests).  sort_free: refined
    levels get their topology from the parent's (phfem_dist_refine_level);
    otherwise every level repeats the occurrence exchange + sort."""
    W = comm.world
    tr = comm.trace = _Trace(states)
    # element ranges: the input split, x4 per refinement (children of [a,b) are [4a,4b))
    esplits = element_splits(nE, W)
    splits, per, (Etot, Btot) = _edge_generation(states, comm, nC, nE, esplits)
    for lvl in range(levels):
        nD, nN = int(states[0].dirichlet.shape[0]), int(states[0].neumann.shape[0])
        ids = _resolve(states, comm, splits, per, nD, nN)
        tr("resolve")
        if sort_free:
            # the last level also produces C's rows (fused, from the parent Neumann edges)
            splits, per, (Etot_f, Btot_f) = _refine_sort_free(states, comm, nC, nE, splits, per, Etot, Btot,
                                                              esplits, nD, nN, ids, fused_c=lvl == levels - 1,
                                                              last=lvl == levels - 1)
        else:
            _refine_sorted(states, comm, nC, splits, per, Etot, nD, nN, ids)
        nC, nE = nC + Etot, 4 * nE
        esplits = 4 * esplits
        if sort_free:
            Etot, Btot = Etot_f, Btot_f
        else:
            splits, per, (Etot, Btot) = _edge_generation(states, comm, nC, nE, esplits)
        tr("refine")
    # final level: the blocks + load first, overlapped with what follows when
    # the backend and communicator allow (side stream; the rest synchronises
    # the host several times)
    overlap = getattr(comm, "overlap_volume", False) and hasattr(states[0].ops, "volume_start")
    for s in states:
        s.mview = s.ops.mesh_view(s.coords, nC, s.elements, s.ehi - s.elo, nE)
        if overlap:
            s.blocks = s.ops.volume_start(s.mview, coeffs, f, t)
    nD, nN = int(states[0].dirichlet.shape[0]), int(states[0].neumann.shape[0])
    ids = _resolve(states, comm, splits, per, nD, nN)
    Ls = []
    for s, (E0, _), i in zip(states, per, ids):
        dl = i[:nD] - E0
        nl = i[nD:] - E0
        E_r = s.ops.num_edges()
        s.dir_local = dl[(dl >= 0) & (dl < E_r) & (i[:nD] >= 0)].to(torch.int32).contiguous()
        own_n = (nl >= 0) & (nl < E_r) & (i[nD:] >= 0)
        s.neu_pos = torch.nonzero(own_n).flatten()
        s.neu_local = nl[own_n].to(torch.int32).contiguous()
        fo = getattr(s, "fine_offsets", None)
        Ls.append(torch.tensor([s.ops.classify(s.dir_local, s.neu_local, E0, fo[1]) if fo else
                                s.ops.classify(s.dir_local, s.neu_local, E0)], dtype=torch.int64,
                               device=s.coords.device))
    tr("classify")
    gl = comm.all_gather(Ls)
    results = []
    for s, (E0, B0), g_ in zip(states, per, gl):
        L_all = torch.stack(g_).flatten().cpu().numpy()
        R0 = int(L_all[:s.rank].sum())
        s.stats = {"E": Etot, "n_boundary": Btot, "L": int(L_all.sum()),
                   "nnz": 4 * int(L_all.sum()) - 2 * (Btot - (Etot - int(L_all.sum())))}
        N0 = E0 - R0                      # Neumann edges before the rank
        nnz0 = 4 * R0 - 2 * (B0 - N0)     # retained boundary rows hold 2 entries
        mview = s.mview
        s.ops.constraint(mview)
        s.bd = s.ops.dirichlet(mview, uD, t)
        fo = getattr(s, "fine_offsets", None)
        if fo is not None:
            assert fo == (E0, R0), (fo, E0, R0)  # the level's offsets == the classification's
        s.ops.rebase_results(E0, R0, nnz0, retained=fo is None, row_ptr=fo is None)
        s.E0, s.R0 = E0, R0
        if not overlap:
            s.blocks = s.ops.volume(mview, coeffs, f, t)
    tr("C+bd+volume")
    # Neumann: owners publish {a, b, t_plus, led}; element owners add b + LN
    all_neu = ids[0][nD:]
    dup = bool(nN) and int(torch.unique(all_neu).numel()) < nN
    tables = [s.ops.neumann_table(s.neu_local, nN, s.neu_pos) for s in states]
    if nN:
        comm.all_reduce(tables, "sum")
    for s, tb in zip(states, tables):
        if overlap:
            s.ops.volume_join()
        s.ops.neumann_apply(s.mview, tb, dup, s.elo, s.ehi, g, t, s.blocks["load"])
    tr("neumann")
    tr.dump()
    comm.trace = None
    return states, nC, nE


def rank_slice(s: RankState) -> dict:
    """One rank's slice of every output (host arrays, global ids)."""
    p = s.ops.part_arrays()
    c = s.ops.cls_arrays()
    rp, col, val = s.ops.csr_arrays()
    out = {k: np.asarray(p[k]) for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus",
                                          "interior_edges", "boundary_edges", "node_edge_start")}
    out["elem_edge"] = s.elem_edge.cpu().numpy()
    out["retained_pos"], out["retained_edges"] = np.asarray(c["retained_pos"]), np.asarray(c["retained_edges"])
    out["C_row_ptr"], out["C_col_idx"], out["C_values"] = np.asarray(rp), np.asarray(col), np.asarray(val)
    out["bd"] = s.bd.cpu().numpy()
    for k in ("B", "D", "M", "M0", "load"):
        out[k] = s.blocks[k].cpu().numpy().reshape(-1)
    if getattr(s, "mid_own", None) is not None:  # after a halo-form last level: parent nodes + owned midpoints
        out["coords_parent"] = s.coords[:s.nc_parent].cpu().numpy()
        out["mid_own"] = s.mid_own.cpu().numpy()
    else:
        out["coords"] = s.coords.cpu().numpy()
    out["elements"] = s.elements.cpu().numpy()
    out["dirichlet"] = s.dirichlet.cpu().numpy()
    out["neumann"] = s.neumann.cpu().numpy()
    return out


def concat_slices(sl: list) -> dict:
    """Rank slices (rank order) -> the single-GPU layout."""
    out = {}
    for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "interior_edges",
              "boundary_edges", "elem_edge", "retained_pos", "retained_edges", "C_col_idx", "C_values", "bd",
              "B", "D", "M", "M0", "load", "elements"):
        out[k] = np.concatenate([x[k] for x in sl])
    out["node_edge_start"] = np.concatenate([x["node_edge_start"][:-1] for x in sl] + [sl[-1]["node_edge_start"][-1:]])
    out["C_row_ptr"] = np.concatenate([x["C_row_ptr"][:-1] for x in sl] + [sl[-1]["C_row_ptr"][-1:]])
    for k in ("dirichlet", "neumann"):
        out[k] = sl[0][k]
    if "mid_own" in sl[0]:
        out["coords"] = np.concatenate([sl[0]["coords_parent"]] + [x["mid_own"] for x in sl])
    else:
        out["coords"] = sl[0]["coords"]
    return out


def collect(states: List[RankState]) -> dict:
    """Rank slices of the emulated ranks concatenated (tests)."""
    return concat_slices([rank_slice(s) for s in states])


def make_states(hm: capi.HostMesh, comm, ops_factory) -> List[RankState]:
    """Replicated input mesh, element ranges split evenly; ops_factory(rank)
    gives the backend of a rank (its device)."""
    es = element_splits(hm.nE, comm.world)
    states = []
    for r in comm.ranks:
        ops = ops_factory(r)
        dev = ops.dev
        states.append(RankState(
            rank=r, ops=ops,
            coords=torch.as_tensor(hm.coords).to(dev).contiguous(),
            elements=torch.as_tensor(hm.elements[es[r]:es[r + 1]]).to(dev).contiguous(),
            elo=int(es[r]), ehi=int(es[r + 1]),
            dirichlet=torch.as_tensor(hm.dirichlet).to(dev).contiguous(),
            neumann=torch.as_tensor(hm.neumann).to(dev).contiguous()))
    return states
