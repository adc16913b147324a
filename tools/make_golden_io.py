"""Generate tests/golden/io/io_golden.npz from the REFERENCE build (oracle/_ref):
save_mesh text and the CLI's topology CSV of the test meshes, and load_mesh's
result (arrays or exception text) for every case of tests/test_io.py.
Run in the container that has /root/reference (the fixture is committed)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import reference as R  # noqa: E402
import test_io as T  # noqa: E402

out = {}
for name, hm in T.io_meshes():
    rm = R.RMesh(hm)
    for w, part in enumerate(R.save_mesh_text(rm)):
        out[f"{name}_save{w}"] = np.frombuffer(part, dtype=np.uint8)
    out[f"{name}_csv"] = np.frombuffer(R.topology_csv(rm), dtype=np.uint8)
for name, c, e, d, n in T.CASES:
    hm, msg = T.ref_load(c, e, d, n)
    if msg is not None:
        out[f"case_{name}_error"] = np.array(msg)
    else:
        for k, x in enumerate(T.arrays(hm)):
            out[f"case_{name}_{k}"] = x
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "io", "io_golden.npz"), **out)
print(len(out), "arrays")
