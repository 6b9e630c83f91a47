"""Host-side selection rules (no GPU): dense vs multifrontal low-order
factors (pmg.use_multifrontal; DESIGN 3 'Selection')."""
import numpy as np
import torch

from paper_2003_02431_b200 import pmg


def test_low_order_factor_selection(monkeypatch):
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda *a, **k: (170 << 30, 180 << 30))
    monkeypatch.delenv("XDG_LOW_ORDER", raising=False)
    assert not pmg.use_multifrontal(np.zeros(0, np.int64))
    # cfg1 / 8^3 p=3-sized Schwarz plans: dense
    assert not pmg.use_multifrontal(np.full(8, 1800))
    # cfg2 level 1: 337 systems of ~1,810 unknowns = 8.8 GB of dense inverses
    assert pmg.use_multifrontal(np.full(337, 1810))
    # 16^3 p=3: 64 systems (1.7 GB)
    assert pmg.use_multifrontal(np.full(64, 1800))
    # one large system (GMRES-PMG global low-order system)
    assert pmg.use_multifrontal(np.array([336_610]))
    assert pmg.use_multifrontal(np.array([16_001]))
    assert not pmg.use_multifrontal(np.array([10_480]))  # cfg2 coarsest: 0.88 GB
    # dense factors must fit: 0.6 of the free memory
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda *a, **k: (1 << 30, 180 << 30))
    assert pmg.use_multifrontal(np.full(40, 1500))  # 0.72 GB > 0.6 GB
    # the switch forces either path
    monkeypatch.setenv("XDG_LOW_ORDER", "dense")
    assert not pmg.use_multifrontal(np.full(337, 1810))
    monkeypatch.setenv("XDG_LOW_ORDER", "sparse")
    assert pmg.use_multifrontal(np.full(2, 10))
