"""The error bound behind predicted compaction (DESIGN.md 5.3,
chains.cu: pred_decide / pk_widen), checked against the reference's own
chains.

A checkpoint's raw concretisation and every constant chain are folds
acc = add_up/add_down(acc, t_j) (interval.hpp:59-96, backsub.hpp:756-759).
The predicted offers replace such a fold by a round-to-nearest parallel sum S
(any order) and claim |fold - (k0 + S)| <= E with

    B = (|k0| + e0 + sum |t_j|) (1 + 2^-30),   E = e0 + 4 (n + 2) (2^-52 B + 2^-1074)

where (k0, e0) is the predicted start value and its radius (e0 = 0 for an
exact start). A row is dropped only when k0 + S + E <= 0 (upper) or
k0 + S - E >= 0 (lower), so a wrong bound could drop a row the reference keeps.
These tests fold adversarial chains with the C restatement of the reference
(oracle/polycert_port.c, pinned to the compiled reference in test_oracle.py)
and compare exactly (fractions). Test infrastructure only.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle.pyoracle import Port


@pytest.fixture(scope="module")
def port():
    return Port()


def ru(x):  # an upper bound of a round-to-nearest result (one step up)
    return math.nextafter(x, math.inf)


def predicted(k0, e0, terms, rng):
    """The device's prediction: an RN sum in an arbitrary order + the radius."""
    t = [x for x in terms if x == x]
    rng.shuffle(t)
    S, A = k0, 0.0
    for x in t:
        S += x
        A += abs(x)
    n = len(t)
    B = ru(ru(ru(abs(k0) + e0) + A) * (1.0 + 2.0**-30))
    E = ru(e0 + ru(4.0 * (n + 2) * ru(ru(2.0**-52 * B) + 2.0**-1074)))
    return S, E


def term_set(rng, n, kind):
    e = rng.randint(-40, 20)
    out = []
    for _ in range(n):
        r = rng.random()
        if kind == "ties":  # multiples of a power of two near the accumulator's ulp
            x = rng.choice([0.5, 1.5, 2.5, 0.25, 3.0]) * 2.0 ** rng.randint(-52, -40)
        elif kind == "wide":
            x = rng.uniform(0.5, 1.0) * 2.0 ** rng.randint(-1074 // 2, 30)
        elif kind == "tiny":
            x = rng.uniform(0.0, 1.0) * 2.0 ** rng.randint(-1074, -1000)
        elif kind == "cancel":
            x = rng.uniform(0.9, 1.1) * 2.0**e
        else:
            x = rng.uniform(0.5, 1.0) * 2.0 ** (e + rng.randint(-30, 5))
        if r < 0.5:
            x = -x
        if r > 0.97:
            x = float("nan")  # a skipped (zero) term
        out.append(x)
    return out


KINDS = ["mixed", "ties", "wide", "tiny", "cancel"]


@pytest.mark.parametrize("kind", KINDS)
def test_single_step_bound(port, kind):
    rng = random.Random(hash(kind) & 0xFFFF)
    chains, length = 300, 200
    acc0 = np.array([rng.choice([0.0, 1.0, -1.0, 2.0**-60, 3.5]) * rng.uniform(0.5, 2.0) for _ in range(chains)])
    terms = np.array([term_set(rng, length, kind) for _ in range(chains)])
    up = np.array([rng.randint(0, 1) for _ in range(chains)], dtype=np.int32)
    v = port.chain_fold(acc0, terms, up)
    for c in range(chains):
        S, E = predicted(float(acc0[c]), 0.0, list(terms[c]), rng)
        assert math.isfinite(v[c])
        assert abs(Fraction(v[c]) - Fraction(S)) <= Fraction(E), (kind, c, v[c], S, E)


def test_bound_chains_across_steps(port):
    """Radii carried through several steps (pk_widen): the prediction of step
    k starts from step k-1's prediction, the reference from its exact fold."""
    rng = random.Random(7)
    chains, steps = 200, 6
    exact = np.array([rng.uniform(-1.0, 1.0) for _ in range(chains)])
    pred = [(float(x), 0.0) for x in exact]
    up = np.array([rng.randint(0, 1) for _ in range(chains)], dtype=np.int32)
    for k in range(steps):
        terms = np.array([term_set(rng, 150, KINDS[k % len(KINDS)]) for _ in range(chains)])
        exact = port.chain_fold(exact, terms, up)
        nxt = []
        for c in range(chains):
            S0, e0 = pred[c]
            S, E = predicted(S0, e0, list(terms[c]), rng)
            assert abs(Fraction(exact[c]) - Fraction(S)) <= Fraction(E), (k, c)
            nxt.append((S, E))
        pred = nxt


def test_decisions_are_sound(port):
    """Near-zero chains: whenever the prediction proves the sign, the
    reference's fold has it (the freeze test of backsub.hpp:814-817)."""
    rng = random.Random(11)
    chains, length = 2000, 64
    acc0 = np.zeros(chains)
    terms = []
    for _ in range(chains):
        t = term_set(rng, length, "cancel")
        # shift the sum close to zero: the cases a loose bound would get wrong
        s = sum(x for x in t if x == x)
        t[0] = -s + rng.uniform(-1e-13, 1e-13) * abs(s) if t[0] == t[0] else t[0]
        terms.append(t)
    terms = np.array(terms)
    up = np.array([rng.randint(0, 1) for _ in range(chains)], dtype=np.int32)
    v = port.chain_fold(acc0, terms, up)
    decided = 0
    for c in range(chains):
        S, E = predicted(0.0, 0.0, list(terms[c]), rng)
        if ru(S + E) <= 0.0:
            decided += 1
            assert v[c] <= 0.0
        if S - E > 0.0 and math.nextafter(S - E, -math.inf) >= 0.0:
            decided += 1
            assert v[c] >= 0.0
    assert decided > 0
