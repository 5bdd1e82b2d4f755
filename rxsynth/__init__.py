"""rxsynth — seeded synthetic transmitter, channel and ADC for the receiver's tests and bench.

TEST / BENCH INFRASTRUCTURE. This module is the one piece shared by the oracle tests and
the CUDA-path tests (task rule: "only the seeded input generators serve both, from a module
of their own"). It holds NO receiver arithmetic: no overlap-save framing, no Kramers-Kronig
reconstruction, no clock recovery, no equaliser, no decision or error counting. It models
only what happens *before* the ADC in the paper's experiments (§III-D
for PAM, §IV-E P:238 for KK-QAM), as SURVEY.md §8(d) restates them, and it designs the
static receiver taps the harness hands to ``rx_create`` (the paper's "optimised offline"
inputs).

Everything is numpy fp64 with ``numpy.random.default_rng(seed)`` (PCG64).
"""
from .gen import (  # noqa: F401
    FS,
    PRBS_PERIOD,
    Record,
    gray,
    gray_inverse,
    kk_record,
    pam_levels,
    pam_record,
    prbs_period_bits,
    qam_axis_levels,
    reference_level_indices,
    static_taps_kk,
    static_taps_pam,
    tile_codes,
)
from .configs import CONFIGS, make_config  # noqa: F401
