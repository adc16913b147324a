"""B200-native edge generation, red refinement and assembly for the lowest-order
primal hybrid FEM (arXiv 2401.15557).

The product is the sm_100a library ``libphfem_b200.so`` behind the C ABI in
``include/phfem_gpu.h``; ``capi`` is its ctypes binding (the Python mirror of
the reference's C++ entry points), ``meshgen`` the seeded BASELINE inputs.
"""
from . import capi, meshgen  # noqa: F401
from .capi import (Context, DeviceMesh, HostMesh, assemble_constraint, assemble_dirichlet,  # noqa: F401
                   assemble_load, assemble_neumann, assemble_volume, build_topology,
                   classify_edges, constraint_csc, load_library, orient_ccw, pipeline, red_refine)
