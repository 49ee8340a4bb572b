"""Host logic of the device density control: the prefix-sum form of the pick
loop (density.py:_decide) equals the reference's sequential loop
(trisplat/density.py:221-245) on random eligibility patterns."""
import numpy as np


def _loop(elig, remaining):
    proc = np.zeros(len(elig), bool)
    split = np.zeros(len(elig), bool)
    for k, e in enumerate(elig):
        if remaining <= 0:
            break
        proc[k] = True
        if e and remaining >= 3:
            split[k] = True
            remaining -= 3
        else:
            remaining -= 1
    return proc, split, remaining


def test_decide_matches_sequential_loop():
    from paper_2505_19175_b200.density import _decide
    rng = np.random.default_rng(0)
    for trial in range(3000):
        k = int(rng.integers(0, 40))
        elig = rng.uniform(0, 1, k) < rng.uniform(0, 1)
        rem = int(rng.integers(1, 3 * k + 3))
        rem = min(rem, max(k, 1)) if trial % 2 else rem
        p, s, r = _decide(elig, rem)
        q, t, u = _loop(elig, rem)
        assert np.array_equal(p, q) and np.array_equal(s, t) and r == u, (elig, rem)
