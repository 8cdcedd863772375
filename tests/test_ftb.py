"""Fraction-to-boundary rule (SPEC fraction_to_boundary): oracle pinned to SPEC's worked
examples and to the defining inequality; the C-ABI kernel bit-exact against it."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.kkt import fraction_to_boundary as ftb


def test_spec_examples():
    assert ftb([1.0, 2.0], [0.5, 3.0], 0.99) == 1.0          # ds >= 0 -> alpha = 1
    assert ftb([1.0], [-1.0], 0.995) == 0.995                 # ratio formula
    assert ftb([1.0, 2.0], [-2.0, 1.0], 0.99) == 0.495        # min over the blocking index
    assert ftb([], [], 0.99) == 1.0


@pytest.mark.parametrize("seed", range(5))
def test_defining_inequality(seed):
    """alpha satisfies s + alpha ds >= (1 - tau) s everywhere, and is the largest such alpha:
    at alpha (1 + 1e-9) some blocking entry violates it (or alpha = 1)."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.uniform(-5, 5, 200))
    ds = rng.standard_normal(200) * np.exp(rng.uniform(-5, 5, 200))
    tau = 0.99
    a = ftb(s, ds, tau)
    assert 0 < a <= 1
    assert np.all(s + a * ds >= (1 - tau) * s * (1 - 1e-12))
    if a < 1:
        b = a * (1 + 1e-9)
        assert np.any(s + b * ds < (1 - tau) * s)


@pytest.mark.gpu
def test_gpu_ftb_bit_exact():
    """ckkt_fraction_to_boundary on a batch (incl. an all-nonnegative row, a NaN entry and a ragged
    length that is not a multiple of the block) equals the oracle bit for bit."""
    import torch
    from paper_2403_15913_b200 import ckkt
    rng = np.random.default_rng(11)
    B, n = 4, 300_001
    s = np.exp(rng.uniform(-8, 8, (B, n)))
    ds = rng.standard_normal((B, n)) * np.exp(rng.uniform(-8, 8, (B, n)))
    ds[1] = np.abs(ds[1])
    ds[2, 17] = np.nan
    dev = torch.device("cuda:0")
    a = ckkt.fraction_to_boundary(torch.as_tensor(s, device=dev), torch.as_tensor(ds, device=dev), 0.995)
    got = a.cpu().numpy()
    for b in range(B):
        assert got[b] == ftb(s[b], ds[b], 0.995), b
    assert got[1] == 1.0
    empty = ckkt.fraction_to_boundary(torch.zeros((2, 0), dtype=torch.float64, device=dev),
                                      torch.zeros((2, 0), dtype=torch.float64, device=dev), 0.99)
    assert empty.cpu().numpy().tolist() == [1.0, 1.0]
