"""B200-native Newton-step hot path of Liu & Marsden's VMS hyper-elastodynamics
scheme (arXiv:1809.06350), drop-in for the reference `elastodyn` library's
assembly / nested block-preconditioned solve / Krylov layer.

The product is ``lib/libelastodyn_b200.so`` (CUDA for sm_100a behind the
C-ABI in ``include/elastodyn_b200.h``); this package is its host-side mirror
of the reference interface.  See DESIGN.md.
"""
from . import _native
from .api import (Context, Csr, ElementInversion, State, Unsupported, amg_options, block_solver_options,
                  compute_tau, dispersed_fiber, fiber_structure_tensors, gen_alpha_scalars, incompressible_neo_hookean, krylov_config,
                  neo_hookean, wave_speed)
from .mesh import Mesh, circumferential_fiber_dirs, generate_box_mesh, generate_cube_mesh, generate_cylinder_mesh
from .problem import CONFIGS, CubeProblem, CylinderProblem

__all__ = [
    "Context", "Csr", "ElementInversion", "State", "Unsupported", "amg_options", "block_solver_options",
    "compute_tau", "dispersed_fiber", "gen_alpha_scalars", "incompressible_neo_hookean", "krylov_config",
    "neo_hookean", "wave_speed", "Mesh", "generate_box_mesh", "generate_cube_mesh", "CONFIGS", "CubeProblem",
    "CylinderProblem", "circumferential_fiber_dirs", "fiber_structure_tensors", "generate_cylinder_mesh",
]


def library_path() -> str:
    return _native.LIB_PATH
