"""TEST INFRASTRUCTURE: a numpy restatement of the per-rank operations of
paper_2401_15557_b200/dist.py (the interface of dist.CudaRankOps), so the
distributed orchestration — key ranges, all-to-alls, id re-basing, boundary
pair resolution, the Neumann table — runs under a real gloo process group on
CPU.  Per-element values come from the C oracle (oracle/), the rest is plain
numpy following the same reference lines as the kernels:
  occurrences / dedup      edge_topology.cpp:52-115
  children / midpoints     refine.cpp:16-37
  refined level            SURVEY §8(f1) closed form (refine.cpp:28-37 +
                           edge_topology.cpp:59-113), the groups of the
                           rank's own parent edges
  classification           edge_topology.cpp:145-177
  C rows                   assembly.cpp:144-168
  Dirichlet / Neumann      assembly.cpp:205-242, elliptic.cpp:54-55
Never used by the product path.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from oracle import oracle as O
from paper_2401_15557_b200 import capi

PI = 3.14159265358979323846


def field_eval(f, x, y, t):
    k, p = f.kind, f.p
    if k == capi.FIELD_ZERO:
        return 0.0
    if k == capi.FIELD_CONST:
        return p[0]
    if k == capi.FIELD_SINSIN:
        return p[0] * math.sin(PI * x) * math.sin(PI * y)
    if k == capi.FIELD_EXP_SINSIN:
        return math.exp(-t) * p[0] * math.sin(PI * x) * math.sin(PI * y)
    if k == capi.FIELD_AFFINE:
        return p[0] + p[1] * x + p[2] * y + p[3] * t
    raise NotImplementedError(k)


def flux_eval(g, x, y, nx, ny, t):
    k, p = g.kind, g.p
    if k == capi.FLUX_ZERO:
        return 0.0
    if k == capi.FLUX_CONST:
        return p[0]
    if k == capi.FLUX_GRAD_SINSIN:
        gx = p[0] * PI * math.cos(PI * x) * math.sin(PI * y)
        gy = p[0] * PI * math.sin(PI * x) * math.cos(PI * y)
        return gx * nx + gy * ny
    raise NotImplementedError(k)


class _Part:
    pass


class NumpyRankOps:
    def __init__(self):
        self.dev = torch.device("cpu")

    def as_tensor(self, a, dtype=torch.int32):
        return torch.as_tensor(np.ascontiguousarray(a)).to(dtype=dtype)

    @staticmethod
    def _dest(splits, v):
        return np.searchsorted(splits, v, side="right") - 1

    # -- edge dedup -------------------------------------------------------------------------
    def occurrences(self, elements, elo, ehi, splits, pack):
        el = elements.numpy().reshape(-1, 3)
        sp = splits.numpy().astype(np.int64)
        n = el.shape[0]
        a = el.reshape(-1)
        b = el[:, [1, 2, 0]].reshape(-1)
        hi, lo = np.maximum(a, b), np.minimum(a, b)
        occ = 3 * (elo + np.repeat(np.arange(n), 3)) + np.tile(np.arange(3), n)
        d = self._dest(sp, hi)
        W = len(sp) - 1
        cnt = np.bincount(d, minlength=W)[:W].astype(np.int32)
        if not pack:
            return torch.as_tensor(cnt)
        order = np.argsort(d, kind="stable")
        rec = np.stack([hi, lo, occ, (a > b).astype(np.int64)], 1)[order].astype(np.int32)
        return torch.as_tensor(rec), cnt.tolist()

    def dedup(self, recv, nlo, nhi, nC, nE, own_range=None):
        r = recv.numpy().astype(np.int64).reshape(-1, 4)
        order = np.lexsort((r[:, 2], r[:, 1], r[:, 0]))   # (max, min, occurrence)
        r = r[order]
        key = r[:, 0] * (nC + 1) + r[:, 1]
        start = np.ones(len(r), bool)
        start[1:] = key[1:] != key[:-1]
        idx = np.flatnonzero(start)
        cnt = np.diff(np.append(idx, len(r)))
        if np.any(cnt > 2):
            raise RuntimeError("non-manifold")
        E = len(idx)
        f = r[idx]
        two = cnt == 2
        g = np.zeros_like(f)
        g[two] = r[idx[two] + 1]
        if np.any(two & (g[:, 3] == f[:, 3])):
            raise RuntimeError("duplicate directed")
        mf, lf = f[:, 2] // 3, (f[:, 2] % 3 + 2) % 3
        mg, lg = g[:, 2] // 3, (g[:, 2] % 3 + 2) % 3
        p = _Part()
        p.edge_nodes = np.where(f[:, 3:4] == 1, f[:, [0, 1]], f[:, [1, 0]]).astype(np.int32)
        p.edge_elements = np.stack([mf, np.where(two, mg, -1)], 1).astype(np.int32)
        p.ltp = lf.astype(np.int32)
        p.ltm = np.where(two, lg, -1).astype(np.int32)
        ids = np.arange(E)
        p.interior = ids[two].astype(np.int32)
        p.boundary = ids[~two].astype(np.int32)
        nodes = np.arange(nlo, nhi + 1)
        p.nes = np.searchsorted(f[:, 0], nodes, side="left").astype(np.int32)
        p.nlo = nlo
        self.part = p
        pairs = np.full((2 * E, 2), -1, np.int32)
        pairs[0::2, 0], pairs[0::2, 1] = 3 * mf + lf, ids
        pairs[1::2, 0] = np.where(two, 3 * mg + lg, -1)
        pairs[1::2, 1] = ~ids
        self.pairs = pairs
        return E, int((~two).sum())

    def refine_level(self, ee_all, el_all, coords, nc, E0p, nlo, nhi, nE_all, neu_parent=None, fine_range=None):
        """Groups of the own parent edges e: the two halves (the one at the
        smaller old node first), then the interior edges mu(e') - mu(e) for the
        partners e' < e of e's elements, ascending e'."""
        p = self.part
        ee = ee_all.numpy().reshape(-1, 3).astype(np.int64)
        ee = np.where(ee >= 0, ee, ~ee)
        c = coords.numpy()
        E = len(p.ltp)
        rows, isb = [], []
        nes = np.zeros(nhi - nlo + 1, np.int32)
        mids = np.zeros((E, 2))
        for le in range(E):
            e = E0p + le
            a, b = (int(x) for x in p.edge_nodes[le])
            tp, tm = (int(x) for x in p.edge_elements[le])
            l = int(p.ltp[le])
            l2 = int(p.ltm[le]) if tm >= 0 else 0
            mu = nc + e
            nes[mu - nlo] = len(rows)
            mids[le] = [0.5 * (c[a][0] + c[b][0]), 0.5 * (c[a][1] + c[b][1])]
            j1, j2, k1, k2 = (l + 1) % 3, (l + 2) % 3, (l2 + 1) % 3, (l2 + 2) % 3
            h1 = (a, mu, 4 * tp + 1 + j1, 2, 4 * tm + 1 + k2 if tm >= 0 else -1, 1 if tm >= 0 else -1)
            h2 = (mu, b, 4 * tp + 1 + j2, 1, 4 * tm + 1 + k1 if tm >= 0 else -1, 2 if tm >= 0 else -1)
            halves = [h1, h2] if a < b else [h2, h1]
            cand = []
            q0, q1 = int(ee[tp][j1]), int(ee[tp][j2])
            if q0 < e:
                cand.append((q0, (mu, nc + q0, 4 * tp, j2, 4 * tp + 1 + j2, 0)))
            if q1 < e:
                cand.append((q1, (nc + q1, mu, 4 * tp, j1, 4 * tp + 1 + j1, 0)))
            if tm >= 0:
                r0, r1 = int(ee[tm][k1]), int(ee[tm][k2])
                if r0 < e:
                    cand.append((r0, (mu, nc + r0, 4 * tm, k2, 4 * tm + 1 + k2, 0)))
                if r1 < e:
                    cand.append((r1, (nc + r1, mu, 4 * tm, k1, 4 * tm + 1 + k1, 0)))
            group = halves + [x for _, x in sorted(cand)]
            rows += group
            isb += [tm < 0, tm < 0] + [False] * (len(group) - 2)
        if E:
            nes[nhi - nlo] = len(rows)
        r = np.asarray(rows, np.int64).reshape(-1, 6)
        Ef = len(r)
        q = _Part()
        q.edge_nodes = r[:, 0:2].astype(np.int32)
        q.edge_elements = r[:, [2, 4]].astype(np.int32)
        q.ltp = r[:, 3].astype(np.int32)
        q.ltm = r[:, 5].astype(np.int32)
        ids = np.arange(Ef)
        b = np.asarray(isb, bool)
        q.interior, q.boundary = ids[~b].astype(np.int32), ids[b].astype(np.int32)
        q.nes, q.nlo = nes, nlo
        self.part = q
        pairs = np.full((2 * Ef, 2), -1, np.int32)
        pairs[0::2, 0], pairs[0::2, 1] = 3 * r[:, 2] + r[:, 3], ids
        pairs[1::2, 0] = np.where(r[:, 4] >= 0, 3 * r[:, 4] + r[:, 5], -1)
        pairs[1::2, 1] = ~ids
        self.pairs = pairs
        return Ef, int(b.sum()), torch.as_tensor(mids)

    # -- refined level, halo form (the ops of dist._refine_sort_free) ------------------------
    def side_records(self, elements, elem_edge, esplits):
        el = elements.numpy().reshape(-1, 3).astype(np.int64)
        ee = elem_edge.numpy().reshape(-1, 3).astype(np.int64)
        sg = ee.reshape(-1)
        e = np.where(sg >= 0, sg, ~sg)
        rec = np.stack([(e << 1) | (sg < 0), ee[:, [1, 2, 0]].reshape(-1), ee[:, [2, 0, 1]].reshape(-1),
                        el.reshape(-1)], 1)
        sp = esplits.numpy().astype(np.int64)
        d = self._dest(sp, e)
        order = np.argsort(d, kind="stable")
        W = len(sp) - 1
        return torch.as_tensor(rec[order].astype(np.int32)), np.bincount(d, minlength=W)[:W].tolist()

    def side_apply(self, recv, E0):
        E = self.num_edges()
        side = np.zeros((2 * max(E, 1), 3), np.int64)
        r = recv.numpy().astype(np.int64).reshape(-1, 4)
        side[2 * ((r[:, 0] >> 1) - E0) + (r[:, 0] & 1)] = r[:, 1:4]
        self._side = side

    def refine_level_side(self, coords, nc, E0p, nlo, nhi, nE_all, coords_fine, neu_parent=None):
        """Groups of the own parent edges from the side records (partners at
        local l+1, l+2 of t_plus / t_minus): two halves (the one at the smaller
        old node first), then the interior edges to mu(e') for partners e' < e,
        ascending e'; rank bytes as the level kernel packs them."""
        p = self.part
        c = coords.numpy()
        cf = coords_fine.numpy()
        sd = self._side
        E = len(p.ltp)
        rows, isb = [], []
        nes = np.zeros(nhi - nlo + 1, np.int32)
        rk = np.zeros(max(E, 1), np.uint8)
        mid = lambda u, v: [0.5 * (u[0] + v[0]), 0.5 * (u[1] + v[1])]
        for le in range(E):
            e = E0p + le
            a, b = (int(x) for x in p.edge_nodes[le])
            tp, tm = (int(x) for x in p.edge_elements[le])
            l = int(p.ltp[le])
            l2 = int(p.ltm[le]) if tm >= 0 else 0
            mu = nc + e
            nes[mu - nlo] = len(rows)
            cf[mu] = mid(c[a], c[b])
            j1, j2, k1, k2 = (l + 1) % 3, (l + 2) % 3, (l2 + 1) % 3, (l2 + 2) % 3
            h1 = (a, mu, 4 * tp + 1 + j1, 2, 4 * tm + 1 + k2 if tm >= 0 else -1, 1 if tm >= 0 else -1)
            h2 = (mu, b, 4 * tp + 1 + j2, 1, 4 * tm + 1 + k1 if tm >= 0 else -1, 2 if tm >= 0 else -1)
            halves = [h1, h2] if a < b else [h2, h1]
            absd = lambda x: int(x) if x >= 0 else ~int(x)
            q0, q1, vop = absd(sd[2 * le][0]), absd(sd[2 * le][1]), int(sd[2 * le][2])
            part = [(q0, q0 < e, (mu, nc + q0, 4 * tp, j2, 4 * tp + 1 + j2, 0), mid(c[b], c[vop])),
                    (q1, q1 < e, (nc + q1, mu, 4 * tp, j1, 4 * tp + 1 + j1, 0), mid(c[vop], c[a]))]
            if tm >= 0:
                r0, r1, vom = absd(sd[2 * le + 1][0]), absd(sd[2 * le + 1][1]), int(sd[2 * le + 1][2])
                part += [(r0, r0 < e, (mu, nc + r0, 4 * tm, k2, 4 * tm + 1 + k2, 0), mid(c[a], c[vom])),
                         (r1, r1 < e, (nc + r1, mu, 4 * tm, k1, 4 * tm + 1 + k1, 0), mid(c[vom], c[b]))]
            else:
                part += [(0, False, None, None), (0, False, None, None)]
            code = 0
            for i, (q, v, _, pm) in enumerate(part):
                if v:
                    code |= sum(1 for (q2, v2, _, _) in part if v2 and q2 < q) << (2 * i)
                    cf[nc + q] = pm   # the partner midpoint (same bits as its owner's)
            rk[le] = code
            cand = sorted((q, row) for q, v, row, _ in part if v)
            group = halves + [x for _, x in cand]
            rows += group
            isb += [tm < 0, tm < 0] + [False] * (len(group) - 2)
        if E:
            nes[nhi - nlo] = len(rows)
        r = np.asarray(rows, np.int64).reshape(-1, 6)
        Ef = len(r)
        q = _Part()
        q.edge_nodes = r[:, 0:2].astype(np.int32)
        q.edge_elements = r[:, [2, 4]].astype(np.int32)
        q.ltp = r[:, 3].astype(np.int32)
        q.ltm = r[:, 5].astype(np.int32)
        ids = np.arange(Ef)
        b = np.asarray(isb, bool)
        q.interior, q.boundary = ids[~b].astype(np.int32), ids[b].astype(np.int32)
        q.nes, q.nlo = nes, nlo
        self.ppart, self.part, self._rk = p, q, rk
        return Ef, int(b.sum())

    def start_records(self, nes_off, psplits):
        p, nes = self.ppart, self.part.nes
        recs = []
        for le in range(len(p.ltp)):
            for m, l in ((p.edge_elements[le][0], p.ltp[le]), (p.edge_elements[le][1], p.ltm[le])):
                if m >= 0:
                    recs.append((3 * int(m) + int(l), int(nes[le + nes_off]), int(self._rk[le])))
        r = np.asarray(recs, np.int64).reshape(-1, 3)
        sp = psplits.numpy().astype(np.int64)
        d = self._dest(sp, r[:, 0] // 3)
        order = np.argsort(d, kind="stable")
        W = len(sp) - 1
        self.ppart = self._rk = None
        return torch.as_tensor(r[order].astype(np.int32)), np.bincount(d, minlength=W)[:W].tolist()

    def start_apply(self, recv, elo, n):
        gs = np.zeros(3 * n, np.int64)
        grk = np.zeros(3 * n, np.int64)
        r = recv.numpy().astype(np.int64).reshape(-1, 3)
        gs[r[:, 0] - 3 * elo] = r[:, 1]
        grk[r[:, 0] - 3 * elo] = r[:, 2]
        return gs, grk

    def children_slots(self, elements, elem_edge, gs, grk, nc, coords_fine, own=(0, 0)):
        el = elements.numpy().reshape(-1, 3).astype(np.int64)
        ee = elem_edge.numpy().reshape(-1, 3).astype(np.int64)
        cf = coords_fine.numpy()
        kids, fee = [], []
        for m in range(len(el)):
            P, sg = el[m], ee[m]
            e = np.where(sg >= 0, sg, ~sg)
            G, R = gs[3 * m:3 * m + 3], grk[3 * m:3 * m + 3]
            for j in range(3):
                if own[0] <= e[j] < own[1]:
                    continue  # the owner's level pass wrote it
                a, b = P[(j + 1) % 3], P[(j + 2) % 3]
                cf[nc + e[j]] = [0.5 * (cf[a][0] + cf[b][0]), 0.5 * (cf[a][1] + cf[b][1])]
            I = []
            for k in range(3):
                jA, jB = (k + 1) % 3, (k + 2) % 3
                jE, jm = (jA, jB) if e[jA] > e[jB] else (jB, jA)
                field = (0 if sg[jE] >= 0 else 2) + (0 if jm == (jE + 1) % 3 else 1)
                I.append(int(G[jE]) + 2 + ((int(R[jE]) >> (2 * field)) & 3))

            def half(j, v):
                a, b = P[(j + 1) % 3], P[(j + 2) % 3]
                i = int(G[j]) + (0 if v == min(a, b) else 1)
                return i if sg[j] >= 0 else ~i
            M0, M1, M2 = nc + e[0], nc + e[1], nc + e[2]
            kids += [[M0, M1, M2], [P[0], M2, M1], [P[1], M0, M2], [P[2], M1, M0]]
            fee += [[I[0], I[1], I[2]], [~I[0], half(1, P[0]), half(2, P[0])],
                    [~I[1], half(2, P[1]), half(0, P[1])], [~I[2], half(0, P[2]), half(1, P[2])]]
        return (torch.as_tensor(np.asarray(kids, np.int64).reshape(-1, 3).astype(np.int32)),
                torch.as_tensor(np.asarray(fee, np.int64).reshape(-1, 3).astype(np.int32)))

    def num_edges(self):
        return len(self.part.ltp)

    def rebase_part(self, E0):
        p = self.part
        p.interior = p.interior + E0
        p.boundary = p.boundary + E0
        p.nes = p.nes + E0
        p.E0 = E0

    def route_pairs(self, E0, esplits, elo=0, ehi=0):
        pr = self.pairs
        pr = pr[pr[:, 0] >= 0].astype(np.int64)
        v = np.where(pr[:, 1] >= 0, pr[:, 1] + E0, ~(~pr[:, 1] + E0))
        sp = esplits.numpy().astype(np.int64)
        d = self._dest(sp, pr[:, 0] // 3)
        W = len(sp) - 1
        order = np.argsort(d, kind="stable")
        send = np.stack([pr[:, 0], v], 1)[order].astype(np.int32)
        return torch.as_tensor(send), np.bincount(d, minlength=W)[:W].tolist()

    def apply_pairs(self, recv, elo, ehi):
        ee = np.zeros(3 * (ehi - elo), np.int32)
        r = recv.numpy()
        ee[r[:, 0] - 3 * elo] = r[:, 1]
        return torch.as_tensor(ee.reshape(-1, 3))

    def resolve(self, pairs, list_base, nlo, E0):
        p = self.part
        pr = pairs.numpy().reshape(-1, 2)
        ids = np.full(len(pr), -1, np.int32)
        err = (1 << 64) - 1
        for i, (a, b) in enumerate(pr):
            hi, lo = max(a, b), min(a, b)
            if hi < nlo or hi >= nlo + len(p.nes) - 1:
                continue
            l, r = p.nes[hi - nlo] - E0, p.nes[hi - nlo + 1] - E0
            e = -1
            for k in range(l, r):
                if min(p.edge_nodes[k]) == lo:
                    e = k
            pos = list_base + i
            if e < 0:
                err = min(err, pos << 2)
            elif p.edge_elements[e, 1] >= 0:
                err = min(err, (pos << 2) | 1)
            else:
                ids[i] = E0 + e
        e64 = np.array([err], dtype=np.uint64).view(np.int64)
        return torch.as_tensor(ids), torch.as_tensor(e64)

    # -- refinement -----------------------------------------------------------------------------
    def midpoints(self, coords):
        c = coords.numpy()
        en = self.part.edge_nodes
        return torch.as_tensor(0.5 * (c[en[:, 0]] + c[en[:, 1]]))

    def children(self, elements, elem_edge, nC):
        el = elements.numpy()
        s = elem_edge.numpy().astype(np.int64)
        mid = nC + np.where(s >= 0, s, ~s)
        p0, p1, p2 = el[:, 0], el[:, 1], el[:, 2]
        m0, m1, m2 = mid[:, 0], mid[:, 1], mid[:, 2]
        kids = np.stack([np.stack([m0, m1, m2], 1), np.stack([p0, m2, m1], 1),
                         np.stack([p1, m0, m2], 1), np.stack([p2, m1, m0], 1)], 1)
        return torch.as_tensor(kids.reshape(-1, 3).astype(np.int32))

    # -- classification / C / vectors -----------------------------------------------------------------
    def classify(self, dir_local, neu_local, E0=0):
        E = self.num_edges()
        neu = np.zeros(E, bool)
        neu[neu_local.numpy()] = True
        rpos = np.full(E, -1, np.int32)
        keep = np.flatnonzero(~neu)
        rpos[keep] = np.arange(len(keep))
        self.cls = {"retained_pos": rpos, "retained_edges": keep.astype(np.int32),
                    "dirichlet": dir_local.numpy().copy()}
        return len(keep)

    def mesh_view(self, coords, nC, elements, nE_local, nE_cols):
        return {"coords": coords.numpy(), "elements": elements.numpy()}

    def constraint(self, mv):
        p, c = self.part, mv["coords"]
        rp, cols, vals = [0], [], []
        for e in self.cls["retained_edges"]:
            a, b = p.edge_nodes[e]
            d = c[b] - c[a]
            ln = math.sqrt(d[0] * d[0] + d[1] * d[1])
            tp, tm = p.edge_elements[e]
            for cc in range(3):
                if cc != p.ltp[e]:
                    cols.append(3 * tp + cc)
                    vals.append(ln * 0.5)
            if tm >= 0:
                for cc in range(3):
                    if cc != p.ltm[e]:
                        cols.append(3 * tm + cc)
                        vals.append(-ln * 0.5)
            rp.append(len(cols))
        self.csr = [np.asarray(rp, np.int32), np.asarray(cols, np.int32), np.asarray(vals, np.float64)]

    def dirichlet(self, mv, uD, t):
        p, c = self.part, mv["coords"]
        bd = np.zeros(len(self.cls["retained_edges"]))
        for e in self.cls["dirichlet"]:
            a, b = p.edge_nodes[e]
            mx, my = 0.5 * (c[a][0] + c[b][0]), 0.5 * (c[a][1] + c[b][1])
            d = c[b] - c[a]
            ln = math.sqrt(d[0] * d[0] + d[1] * d[1])
            pos = self.cls["retained_pos"][e]
            if pos >= 0:
                bd[pos] = -ln * field_eval(uD, mx, my, t)
        return torch.as_tensor(bd)

    def volume(self, mv, coeffs, f, t):
        hm = capi.HostMesh(mv["coords"], mv["elements"], np.zeros((0, 2)), np.zeros((0, 2)))
        B, D, M, M0 = O.assemble_volume(hm, coeffs)
        load = O.assemble_load(hm, f, t)
        return {"B": torch.as_tensor(B.reshape(-1, 9)), "D": torch.as_tensor(D.reshape(-1, 9)),
                "M": torch.as_tensor(M.reshape(-1, 9)), "M0": torch.as_tensor(M0.reshape(-1, 9)),
                "load": torch.as_tensor(load.reshape(-1, 3).copy())}

    def neumann_table(self, neu_local, nN_all, positions):
        p = self.part
        tab = np.zeros((nN_all, 4), np.int32)
        for pos, e in zip(positions.numpy(), neu_local.numpy()):
            tab[pos] = [p.edge_nodes[e][0], p.edge_nodes[e][1], p.edge_elements[e][0], p.ltp[e]]
        return torch.as_tensor(tab)

    def neumann_apply(self, mv, table, dup, elo, ehi, g, t, load):
        c = mv["coords"]
        ln_acc = {}
        for a, b, tp, led in table.numpy():
            if not (elo <= tp < ehi):
                continue
            mx, my = 0.5 * (c[a][0] + c[b][0]), 0.5 * (c[a][1] + c[b][1])
            dx, dy = c[b][0] - c[a][0], c[b][1] - c[a][1]
            ln = math.sqrt(dx * dx + dy * dy)
            val = flux_eval(g, mx, my, dy / ln, -dx / ln, t)
            acc = ln_acc.setdefault(tp, [0.0, 0.0, 0.0])
            for cc in range(3):
                acc[cc] += ln * val * (0.0 if cc == led else 0.5)
        L = load.numpy()
        for tp, acc in ln_acc.items():
            for cc in range(3):
                L[tp - elo, cc] = L[tp - elo, cc] + acc[cc]

    def rebase_results(self, E0, R0, nnz0, retained=True, row_ptr=True):
        assert retained and row_ptr  # this backend has no count / run level: offsets are always applied here
        rp = self.cls["retained_pos"]
        self.cls["retained_pos"] = np.where(rp >= 0, rp + R0, -1).astype(np.int32)
        self.cls["retained_edges"] = self.cls["retained_edges"] + E0
        self.csr[0] = self.csr[0] + nnz0

    # -- results --------------------------------------------------------------------------------------
    def part_arrays(self):
        p = self.part
        return {"edge_nodes": p.edge_nodes, "edge_elements": p.edge_elements, "local_in_tplus": p.ltp,
                "local_in_tminus": p.ltm, "interior_edges": p.interior, "boundary_edges": p.boundary,
                "node_edge_start": p.nes}

    def cls_arrays(self):
        return {"retained_pos": self.cls["retained_pos"], "retained_edges": self.cls["retained_edges"]}

    def csr_arrays(self):
        return tuple(self.csr)

    def release(self):
        pass
