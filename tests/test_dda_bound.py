"""The int32 bound of the walk's decision terms (k_id.cu header), checked on
the formulation itself (CPU, no GPU): the pairwise terms q_ab = floor((N_a |D_b| - N_b |D_a| - bias)/S)
with S = 65536 (Q16), stepped by the sign rule of dda.cuh, (1) stay inside [-|D_a| - 1, |D_b|] at
every step, including K = 16 speculative steps past the ray's end, and (2) visit exactly the voxels
of the oracle's walk (which compares int128 cross products, a different formulation).  Together these
are what make the int32 instance exact for |D| < 2^30 - 1 and identical to the oracle."""
import numpy as np
import pytest

import oracle
from nbt_inputs import random_segments_q16, tie_segments_q16

S = 65536
K = 16


def q_walk(o, e, extra=K):
    """Voxels of the q-term walk of dda.cuh (python ints), and the largest bound violation."""
    D = [int(e[a]) - int(o[a]) for a in range(3)]
    neg = [d < 0 for d in D]
    ad = [abs(d) for d in D]
    v = [int(o[a]) // S for a in range(3)]
    ve = [int(e[a]) // S for a in range(3)]
    n = sum(abs(ve[a] - v[a]) for a in range(3))
    N = [(int(o[a]) - v[a] * S) if neg[a] else ((v[a] + 1) * S - int(o[a])) for a in range(3)]

    def bias(a, b):          # 0 if a moves - and b moves + (then b wins a tie), else 1
        return 0 if (neg[a] and not neg[b]) else 1

    q = {(0, 1): (N[0] * ad[1] - N[1] * ad[0] - bias(0, 1)) // S,
         (0, 2): (N[0] * ad[2] - N[2] * ad[0] - bias(0, 2)) // S,
         (1, 2): (N[1] * ad[2] - N[2] * ad[1] - bias(1, 2)) // S}
    lo = {k: -ad[k[0]] - 1 for k in q}
    hi = {k: ad[k[1]] for k in q}
    worst = 0
    visits = [tuple(v)]
    for s in range(n + extra):
        x_first = q[(0, 1)] < 0 and q[(0, 2)] < 0
        y_first = (not x_first) and q[(1, 2)] < 0
        if x_first:
            q[(0, 1)] += ad[1]; q[(0, 2)] += ad[2]; a = 0
        elif y_first:
            q[(0, 1)] -= ad[0]; q[(1, 2)] += ad[2]; a = 1
        else:
            q[(0, 2)] -= ad[0]; q[(1, 2)] -= ad[1]; a = 2
        for k, val in q.items():
            worst = max(worst, lo[k] - val, val - hi[k])
        v[a] += -1 if neg[a] else 1
        if s < n:
            visits.append(tuple(v))
    return visits, worst


def _all_free(n=8):
    return oracle.OracleMap(np.ones((n, n, n), np.uint8))


@pytest.mark.parametrize("kind", ["random", "ties"])
def test_q_terms_stay_in_bounds_and_match_the_oracle_walk(kind):
    m = _all_free()
    if kind == "random":
        o, e = random_segments_q16(400, -6.0, 14.0, seed=71)
    else:
        o, e = tie_segments_q16(400, 9, seed=72)
        o = o - S
    for oo, ee in zip(o, e):
        visits, worst = q_walk(oo, ee)
        assert worst <= 0, (oo, ee, worst)
        ijk, _, r = oracle.trace_ray(m, oo, ee, max_visits=4096)
        assert visits == [tuple(int(t) for t in x) for x in ijk]


def test_q_terms_bound_on_long_rays():
    """Long walks (up to ~1500 steps) with shallow and steep slopes: the bound holds at every step,
    so the largest |q| is max |D| + 1 regardless of the ray length (no growth with L)."""
    rng = np.random.default_rng(5)
    for _ in range(30):
        o = rng.integers(0, 8 * S, 3)
        d = rng.normal(size=3)
        d[int(rng.integers(0, 3))] *= rng.choice([0.01, 1.0, 30.0])
        d /= np.abs(d).max()
        e = o + np.round(d * rng.uniform(100, 600) * S).astype(np.int64)
        visits, worst = q_walk(o, e)
        assert worst <= 0
        assert len(visits) == 1 + sum(abs(int(e[a]) // S - int(o[a]) // S) for a in range(3))
