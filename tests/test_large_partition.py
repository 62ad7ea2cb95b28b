"""Host-only checks of the large-fleet work partition (st_large_partition): units cover every
agent pair at every sample exactly once, GPUs get contiguous cost-balanced agent-pair ranges,
and every GPU runs one CTA per SM (>= 100 CTAs) at any G up to 8."""

import numpy as np
import pytest

SMS = 148  # B200


def _pairs_of_units(n, part):
    """pair-samples covered by each unit (full lanes x steps, masking partial blocks)."""
    from math import comb
    nb = (n + 31) // 32
    ab = [(a, b) for a in range(nb) for b in range(a, nb)]
    out = np.zeros(part["units"], dtype=np.int64)
    for k, (A, B) in enumerate(ab):
        nA, nB = min(32, n - 32 * A), min(32, n - 32 * B)
        u0, u1 = part["ab_first"][k], part["ab_first"][k + 1]
        out[u0:u1] = comb(nA, 2) if A == B else nA * nB // 2
    return out


@pytest.mark.parametrize("n,m", [(256, 100), (200, 100), (96, 60), (65, 40)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_partition_covers_all_pairs_contiguously(n, m, G):
    from paper_2011_04240_b200 import native
    part = native.large_partition(n, m, G, SMS)
    ur = part["u_range"]
    assert ur[0] == 0 and ur[-1] == part["units"] and np.all(np.diff(ur) >= 0)
    per_unit = _pairs_of_units(n, part)
    assert per_unit.sum() == n * (n - 1) // 2 * m  # every pair at every sample, once
    cost = np.concatenate([[0], np.cumsum(part["rows"])])
    gcost = np.diff(cost[ur])
    assert gcost.max() - gcost.min() <= 2 * 16  # balanced to a unit
    for g in range(G):
        cf = part["cta_first"][g]
        assert cf[0] == ur[g] and cf[-1] == ur[g + 1] and np.all(np.diff(cf) >= 0)
        ccost = np.diff(cost[cf])
        assert ccost.max() - ccost.min() <= 2 * 16


def test_every_gpu_runs_a_full_grid_at_eight_gpus():
    from paper_2011_04240_b200 import native
    part = native.large_partition(256, 100, 8, SMS)
    per_gpu_units = np.diff(part["u_range"])
    assert np.all(per_gpu_units >= SMS)  # >= 1 unit per CTA: all 148 CTAs of every GPU busy
    assert part["cta_first"].shape == (8, SMS + 1)
