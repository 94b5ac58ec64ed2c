"""Seeded synthetic inputs for the five BASELINE.json configs.

Shared by the oracle tests and the CUDA path's tests/bench: it holds NONE of the
Newton–Schulz arithmetic (no sign, no iteration, no reflector) -- only the
recipes that draw spectra, orthogonal factors and the Allen–Cahn Hessian, as
read in DESIGN.md §Inputs.
"""
from .configs import (  # noqa: F401
    cfg0_controlled, cfg1_batched, cfg2_allen_cahn, cfg3_dense, cfg4_sharded,
    householder_spectrum, householder_form_numpy, householder_form_fast, haar_q, rotated_quartic_scan,
)
