"""B200-native stochastic conservative field transfer (arXiv 2603.00538, MC operator).

Drop-in for the reference ``tritransfer`` Monte-Carlo path: meshes, nodal fields,
sample plans, ``assemble_load_mc``, ``transfer_mc``, ``MCTransferOperator``, the
uniform-grid locator, the P1 mass matrix / PCG and conservation reporting -- with
every numeric step running in hand-written sm_100a CUDA (libtt_b200.so) and no CPU
fallback.  Extends the reference (2-D triangles) to 3-D tetrahedra.
"""

from .errors import (CoverageGap, DegenerateElement, DeviceUnavailable, DimensionMismatch, EmptyMesh,
                     InvalidDensity, InvalidParameter, MeshMismatch, NoConvergence,
                     NonManifold, ParseError, SourceEvalFailed, TransferError,
                     ZeroDenominator)
from .mesh import (SimplexMesh, TetMesh, TriMesh, build_adjacency, generate_cube_mesh,
                   generate_square_mesh, generate_torus_mesh, load_msh, save_msh)
from .fem import (NodalField, SparseSymMatrix, assemble_mass_matrix, basis_integrals,
                  cg_solve, integrate_field)
from .locate import EPS_LOC, OUTSIDE, UniformGridLocator
from .montecarlo import (AnalyticField, MeshBackedField, SamplePlan, assemble_load_mc,
                         assemble_load_mc_weighted, bary_map, importance_weights)
from .fields import NAMED_FIELDS, get_field, parse_field
from .transfer import CouplingStep, MCTransferOperator, transfer_mc
from .metrics import (ErrorReport, IntersectionSet, dof_l2_error, find_intersections, mass_error,
                      mesh_mass_error, supermesh_l2_error, supermesh_mass_error)

kernel_backend = "cuda-sm_100a"

__all__ = [
    "TriMesh", "TetMesh", "SimplexMesh", "NodalField", "SparseSymMatrix",
    "generate_square_mesh", "generate_cube_mesh", "generate_torus_mesh", "load_msh", "save_msh", "build_adjacency",
    "assemble_mass_matrix", "cg_solve", "integrate_field", "basis_integrals",
    "UniformGridLocator", "EPS_LOC", "OUTSIDE",
    "AnalyticField", "MeshBackedField", "SamplePlan", "assemble_load_mc",
    "assemble_load_mc_weighted", "importance_weights", "bary_map",
    "NAMED_FIELDS", "get_field", "parse_field",
    "MCTransferOperator", "transfer_mc", "CouplingStep",
    "ErrorReport", "dof_l2_error", "mesh_mass_error", "mass_error", "IntersectionSet",
    "find_intersections", "supermesh_l2_error", "supermesh_mass_error", "CoverageGap",
    "kernel_backend",
]

__version__ = "0.1.0"
