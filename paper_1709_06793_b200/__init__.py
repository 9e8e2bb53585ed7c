"""B200-native stencil-scaling operators for -div(k grad u) = f on HHG
macro-tetrahedra (arXiv 1709.06793), drop-in for the reference `hhgscale`
Operator / GridHierarchy / solve entry points.

Host setup (mesh numbering, reference stencils) is numpy; every operator
application, residual, smoothing sweep and solver vector update runs in the
sm_100a kernels of libhhg_b200.so (csrc/), called through its C ABI
(include/hhg_b200.h).
"""
from .coefficients import (CoefficientField, TensorCoefficient, catalog, kmin_field,
                           sample_nodal)
from .costmodel import analytic_count, traffic
from .mesh import (DIRS_3D, MacroMesh, PrimitiveKind, RefinedGrid,
                   SimplexLattice, cylinder_shell_box, kuhn_blocks,
                   lattice_elements, load_macro_mesh, reference_simplex,
                   refine_uniform, unit_cube_12, unit_cube_6, unit_cube_blocks)
from .operators import VARIANTS, Operator, parse_hybrid_set

__version__ = "0.1.0"

__all__ = [
    "CoefficientField", "TensorCoefficient", "catalog", "kmin_field", "sample_nodal",
    "analytic_count", "traffic", "DIRS_3D", "MacroMesh", "PrimitiveKind",
    "RefinedGrid", "SimplexLattice", "cylinder_shell_box", "kuhn_blocks",
    "lattice_elements", "load_macro_mesh", "reference_simplex",
    "refine_uniform", "unit_cube_12", "unit_cube_6", "unit_cube_blocks",
    "VARIANTS", "Operator", "parse_hybrid_set",
]
