"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref: the
reference's own sources compiled against shim/Eigen).  Run here, where
/root/reference exists; the fixtures travel with the repo to the GPU box.

  python tools/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (mesh refinement for the inputs only)
from oracle import reference as R  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

CASES = {
    "crisscross_L1_cfg2": (lambda: O.refine_levels(G.crisscross_square(), 1), 2),
    "config1_square_L3": (lambda: O.refine_levels(G.square_2tri(), 3), 1),
    "config2_lshape_L2": (lambda: O.refine_levels(G.lshape_6tri(), 2), 2),
    "config3_square_L2": (lambda: O.refine_levels(G.square_2tri(), 2), 3),
    "config4_stress_L3": (lambda: O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 3), 3)), 4),
}


def flat(prefix, d, out):
    for k, v in d.items():
        out[f"{prefix}{k}"] = v


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (mk, cfg) in CASES.items():
        hm = mk()
        coeffs, f, g, uD = G.config_fields(cfg)
        r = R.all_outputs(hm, coeffs, f, g, uD, t=0.0)
        z = {"in_coords": hm.coords, "in_elements": hm.elements, "in_dirichlet": hm.dirichlet,
             "in_neumann": hm.neumann, "cfg": np.array(cfg)}
        flat("topo_", r["topo"], z)
        flat("cls_", r["cls"], z)
        for k in ["B", "D", "M", "M0", "b", "ln", "bd"]:
            z[k] = r[k]
        for k, arr in zip(["outer", "inner", "values"], r["C_csc"]):
            z["csc_" + k] = arr
        for k, arr in zip(["row_ptr", "col_idx", "values"], r["C_csr"]):
            z["csr_" + k] = arr
        fm = r["refined"]
        z.update({"ref_coords": fm.coords, "ref_elements": fm.elements, "ref_dirichlet": fm.dirichlet,
                  "ref_neumann": fm.neumann})
        if cfg == 3:  # CN right-hand side of solve_parabolic, steps 0 and 5
            rm = R.RMesh(hm)
            rt = R.RTopology(rm)
            rc = R.RClassification(rt, rm)
            W = G.uniform_pm1(5, 3 * hm.nE + rc.L)
            z["cn_state"] = W
            z["cn_rhs_0"] = R.cn_rhs(rm, rt, rc, coeffs, f, g, uD, 1e-3, 0, W)
            z["cn_rhs_5"] = R.cn_rhs(rm, rt, rc, coeffs, f, g, uD, 1e-3, 5, W)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **z)
        print(name, hm.nE, "triangles")


if __name__ == "__main__":
    main()
