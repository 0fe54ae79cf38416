"""The windowed / banded oracle used for full-size parity equals the full-frame oracle
bitwise (receptive field covered by the margin; P13/P14 applied to the c1 network)."""
import numpy as np
import pytest

import synth
from helpers import band_oracle, oracle_full, weights_for, window_oracle


@pytest.fixture(scope="module")
def c1_frame():
    cfg = synth.Config("w", 208, 96, 1, 8, 4, (32, 64, 128, 256), 64, "bf16")
    w = weights_for(cfg)
    fr = synth.gen_frames(cfg)
    return cfg, w, fr, oracle_full(cfg, w, fr)


@pytest.mark.parametrize("margin", [40, 64])
def test_window_oracle_bitwise_c1_net(c1_frame, margin):
    cfg, w, _, full = c1_frame
    for rows, cols in (((96, 112), (40, 56)), ((0, 8), (0, 16)), ((200, 208), (80, 96)), ((56, 64), (0, 96))):
        win = window_oracle(cfg, w, 0, rows, cols, margin=margin)
        assert np.array_equal(win, full[rows[0]:rows[1], cols[0]:cols[1]]), (margin, rows, cols)


def test_band_oracle_bitwise_c1_net(c1_frame):
    """The banded, threaded full-frame oracle (margin 40, 24-row bands) = the full oracle."""
    cfg, w, fr, full = c1_frame
    assert np.array_equal(band_oracle(cfg, w, fr, margin=40, threads=4, band=24), full)
