"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/glassnet.h
declares, validates dims synchronously, and fails loudly without a GPU (no CPU path)."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from paper_2405_19056_b200 import glassnet as gb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "glassnet.h")).read()
    return sorted(set(re.findall(r"\b(glassnet_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = gb.lib()
    declared = _declared()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(declared) == sorted(gb.EXPORTS)


@pytest.mark.parametrize("cfg,count", [("c0", 50700), ("c1", 787340)])
def test_weight_count(cfg, count):
    c = synth.CONFIGS[cfg]
    d = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels, precision=c.precision)
    assert gb.weight_count(d) == count == synth.weight_count(c.widths, c.levels, c.t_hidden)


def test_dims_validation_messages():
    d = gb.make_dims(60, 64, 8, (32, 64, 128, 256), 64)      # 60 not a multiple of 8
    assert gb.weight_count(d) == 0
    assert "multiples of 2^(levels-1)" in gb.lib().glassnet_last_error().decode()
    d = gb.make_dims(64, 64, 17, (32, 64, 128, 256), 64)
    assert gb.weight_count(d) == 0
    assert "k_slots > 16" in gb.lib().glassnet_last_error().decode()


def test_tile_rows_rule():
    """units of u = 2^(L-1); rank r gets [floor(rU/N), floor((r+1)U/N))."""
    c = synth.CONFIGS["c4"]
    d = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels)
    assert [gb.tile_rows(d, 2, r) for r in range(2)] == [(0, 1080), (1080, 1080)]
    rows = [gb.tile_rows(d, 4, r)[1] for r in range(4)]
    assert rows == [536, 544, 536, 544]
    t8 = [gb.tile_rows(d, 8, r) for r in range(8)]
    assert sum(n for _, n in t8) == 2160 and all(n in (264, 272) for _, n in t8)
    assert all(t8[i][0] + t8[i][1] == t8[i + 1][0] for i in range(7))


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = synth.CONFIGS["c0"]
    d = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels, precision="fp32")
    w = synth.make_weights(c.widths, c.levels, c.t_hidden)
    with pytest.raises(gb.GlassNetError) as ei:
        gb.GlassNet(w, d)
    assert ei.value.code == 3 and "no CPU path" in str(ei.value)


def test_create_rejects_wrong_weight_count():
    c = synth.CONFIGS["c0"]
    d = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels, precision="fp32")
    with pytest.raises(gb.GlassNetError) as ei:
        gb.GlassNet(np.zeros(10, np.float32), d)
    assert ei.value.code == 1 and "n_weights" in str(ei.value)
