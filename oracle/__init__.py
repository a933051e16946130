"""FP64 CPU oracle for FRAM / SDSN (arXiv 2508.00887) — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA path
(`paper_2508_00887_b200/`, `libfram.so`) is checked against.  It shares no code
with the CUDA path: no kernels, headers, helpers, constants or table
generators.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product path never
routes through it and never falls back to it.

Citation keys: `P:n` = /root/reference/PAPER.md line n (LaTeX source of the
paper); `S:n` = SPEC.md line n; `R<k>` = a reading of a silent/ambiguous point,
listed in DESIGN.md §3 (taken from SURVEY.md §8(c)).

Parity status of every public function is stated in its docstring; functions
without an independent pin say "parity unpinned" (there are none at present —
see DESIGN.md §3.3 for the pin table).
"""

from .fram_oracle import (  # noqa: F401
    DataError,
    precondition,
    gradient,
    p1_project,
    p2_nonneg,
    p3_project,
    gamma,
    sdsn,
    sdsn_fp32,
    dsn_fixed,
    fram,
    objective,
    objective_perm,
    matching_error,
    node_accuracy,
    unary_from_features,
    pad_attributed,
    fram_attributed,
)
from .lap import lap_max, brute_force_max, perm_score  # noqa: F401
from .exact import dykstra_project, affine_projection_kkt, qap_brute_force  # noqa: F401
from .rounding import round_bf16, round_fp16, round_tf32  # noqa: F401
