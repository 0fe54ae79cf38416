"""The windowed oracle used for sampled full-size parity equals the full-frame oracle
bitwise (receptive field covered by the margin; P13/P14 applied to the c1 network)."""
import numpy as np

import synth
from helpers import oracle_full, weights_for, window_oracle


def test_window_oracle_bitwise_c1_net():
    cfg = synth.Config("w", 208, 96, 1, 8, 4, (32, 64, 128, 256), 64, "bf16")
    w = weights_for(cfg)
    full = oracle_full(cfg, w, synth.gen_frames(cfg))
    for rows, cols in (((96, 112), (40, 56)), ((0, 8), (0, 16)), ((200, 208), (80, 96))):
        win = window_oracle(cfg, w, 0, rows, cols, margin=64)
        assert np.array_equal(win, full[rows[0]:rows[1], cols[0]:cols[1]]), (rows, cols)
