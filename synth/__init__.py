"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

Data only: this package holds none of the method's arithmetic (no preconditioning,
gradient, SDSN, update or LAP).  Every recipe is stated in DESIGN.md §4 and stands in
for the paper's datasets (VGG affine, CMU House, SNAP Facebook-ego, UBC), which are
not available.
"""
from .graphs import (  # noqa: F401
    Instance,
    config_c1,
    config_c2,
    config_c3_instance,
    config_c3_batch,
    config_c4,
    config_c5,
    config_ubc,
    ba_graph,
    er_graph,
    random_nonneg,
    random_perm_matrix,
    SCHEDULES,
)
