"""B200-native nodal-DG Maxwell operator (arXiv 0901.1024), drop-in for simtdg's hot path.

Setup mirrors ``simtdg`` (refelem / mesh / maxwell); the RHS and the LSRK4
stage run as hand-written sm_100a kernels in libdgm.so behind a C ABI
(include/dgm.h).  See DESIGN.md.
"""

from .maxwell import (VACUUM, CavityMode, Material, field_energy, flux, l2_error, pec_boundary, stable_dt,
                      upwind_flux)
from .mesh import (VERTEX_PERMUTATIONS, FaceConnectivity, GeometricFactors, Mesh, MeshFormatError,
                   NonConformingMeshError, build_connectivity, compute_geometry, element_inradii,
                   generate_box_mesh, map_nodes, read_tetgen)
from .refelem import (FACE_AREAS, FACE_UNIT_NORMALS, FACE_VERTEX_IDS, NUM_FACES, REFERENCE_VERTICES,
                      ReferenceElement, build_reference_element, face_node_permutation, simplex_node_count)
from .stepper import RK_A, RK_B, RK_C, rk4_step

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so the setup layer imports without CUDA
    if name in ("B200MaxwellOperator", "build_b200_operator"):
        from . import operator

        return getattr(operator, name)
    if name in ("run_cavity", "CavityRun", "UnstableRunError"):
        from . import driver

        return getattr(driver, name)
    if name == "HostStepper":
        from . import hoststep

        return hoststep.HostStepper
    if name in ("build_face_maps", "FaceMaps"):
        from . import facemaps

        return getattr(facemaps, name)
    raise AttributeError(name)


__all__ = [
    "VACUUM", "CavityMode", "Material", "field_energy", "flux", "l2_error", "pec_boundary", "stable_dt",
    "upwind_flux", "VERTEX_PERMUTATIONS", "FaceConnectivity", "GeometricFactors", "Mesh", "MeshFormatError",
    "NonConformingMeshError", "build_connectivity", "compute_geometry", "element_inradii", "generate_box_mesh",
    "map_nodes", "read_tetgen", "FACE_AREAS", "FACE_UNIT_NORMALS", "FACE_VERTEX_IDS", "NUM_FACES",
    "REFERENCE_VERTICES", "ReferenceElement", "build_reference_element", "face_node_permutation",
    "simplex_node_count", "RK_A", "RK_B", "RK_C", "rk4_step", "B200MaxwellOperator", "build_b200_operator",
    "build_face_maps", "FaceMaps", "run_cavity", "CavityRun", "UnstableRunError", "HostStepper",
]
