"""Paper-printed values (tests/golden/paper_values.json, each cited) against the oracle's
constants and arithmetic."""
import json
import math
import os

import numpy as np

from oracle import rx_oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_geometry_constants():
    assert O.N_FFT == G["fft_size"]["value"]
    assert O.HOP == G["valid_per_block"]["value"]
    assert O.HOP * G["blocks_per_buffer"]["value"] == G["buffer_samples"]["value"]
    assert abs(G["buffer_samples"]["value"] / 4e9 * 1e3 - G["buffer_ms_at_4GSa"]["value"]) < 5e-4
    assert 2 * 52 + 1 == G["clock_avg_blocks"]["value"]
    # Hermitian half of the spectrum over a buffer: 512 complex mults/block, 2 per thread
    assert G["blocks_per_buffer"]["value"] * 512 // 2 == G["fd_eq_threads"]["value"]
    # both static filters fit the 100% overlap-save constraint (A3: L odd, L <= hop + 1)
    for k in ("pam_static_taps", "kk_static_taps"):
        O.zero_phase_spectrum(np.ones(G[k]["value"]))


def test_clock_cliff_arithmetic():
    """an 8-bit counter of samples slipped per buffer overflows at 30.5 ppm = 122 kHz."""
    c = G["clock_cliff"]
    slip = G["buffer_samples"]["value"] * c["ppm"] * 1e-6
    assert 2 ** (c["counter_bits"] - 1) - 1 < slip < 2 ** (c["counter_bits"] - 1) + 1
    assert abs(c["ppm"] * 1e-6 * c["adc_gsa"] * 1e9 / 1e3 - c["khz"]) < 0.1


def test_fec_thresholds_and_unwrap_example():
    from scipy.special import erfc
    for q in G["hdfec_q_db"].values():
        if isinstance(q, float):
            ber = 0.5 * erfc(10 ** (q / 20) / math.sqrt(2))
            assert abs(O.q_from_ber(ber) - q) < 1e-9
    ex = G["unwrap_example"]
    ck = O.clock_phase(np.exp(1j * np.array(ex["wrapped"])), half=0)
    assert np.allclose(ck["theta_u"], ex["unwrapped"], atol=1e-12)


def test_carrier_dds_increment_from_paper_frequency():
    f = G["carrier_ghz"]["value"] * 1e9
    inc = O.dds_increment(-f, 4e9)
    assert abs((inc - 2 ** 64) / 2 ** 64 + f / 4e9) < 1e-15
