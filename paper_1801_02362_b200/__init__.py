"""B200-native (sm_100a) aligned-MSD / path-CV / floating-close-structure hot path
of arXiv 1801.02362, drop-in for the reference package's metadyn_close API.

Modules mirroring the reference / SPEC interface:
  geometry (Structure, center, RotationFit, jacobi_eigh, kearsley_fit, rotation_derivative_check)
  msd      (DistanceResult, CloseStructureState, exact_distance, approx_distance,
            step_close_structure, step_original)
  colvar   (ReferenceSet, CVResult, property_map)
  errors   (the reference exception taxonomy)
Batched device entry points: engine (PathCV, msd_matrix, path_cv, close_structure_replay).
All arithmetic runs in libmcb200.so (csrc/, C ABI in include/mcb200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
