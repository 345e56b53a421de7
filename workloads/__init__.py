"""Seeded synthetic inputs for the reordering hot path (shared by tests, bench, smoke).

This package holds NO arithmetic of the method: it only draws random Schur
forms, orthogonal matrices and selections with a counter-based generator.
Both the oracle (``oracle/``) and the product (``paper_1905_04975_b200``)
are fed from here; neither imports the other.
"""
from .schur_inputs import (CONFIGS, Hessenberg, Pencil, Problem, make_config, make_hessenberg,  # noqa: F401
                           make_pencil, make_problem, shift_pairs)
