"""GPU trace generator, host side (no GPU): the integer-exact restatement in
oracle/tracegen_ref.py (the algorithm the CUDA kernel implements) pinned
stage by stage against numpy 2.3 itself -- SeedSequence.spawn pools and
generate_state, PCG64 state and raw output, the recovered exponential
ziggurat tables over 10^6 draws (the rejection path ~10^4 times), Python's
round(t, 6) -- and end to end against the reference's gen_zipf
(workload.py:82-111)."""

from __future__ import annotations

import random

import numpy as np
import pytest

from oracle import tracegen_ref as tr
from paper_2507_08954_b200.workload import default_profiles, gen_zipf, zipf_rates


def _tables():
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "paper_2507_08954_b200", "data", "zig_exp.npz"))
    return [int(v) for v in z["ke"]], [float(v) for v in z["we"]], [float(v) for v in z["fe"]]


@pytest.mark.parametrize("seed", [0, 1, 7, 2 ** 31 + 3, 2 ** 32, 2 ** 40 + 5, 2 ** 64 - 1])
def test_seed_sequence_and_pcg64(seed):
    kids = np.random.SeedSequence(seed).spawn(6)
    for k, kid in enumerate(kids):
        pool = tr.seed_pool(seed, (k,))
        assert pool == [int(x) for x in kid.pool]
        assert tr.generate_state64(pool, 4) == [int(x) for x in kid.generate_state(4, np.uint64)]
        ref = np.random.PCG64(np.random.SeedSequence(seed).spawn(6)[k])
        st = ref.state["state"]
        mine = tr.PCG64(pool)
        assert (mine.state, mine.inc) == (st["state"], st["inc"])
        assert [mine.next64() for _ in range(64)] == ref.random_raw(64).tolist()


def test_ziggurat_tables_replay_numpy():
    ke, we, fe = _tables()
    raw = iter(np.random.PCG64(2024).random_raw(3_000_000).tolist())

    class Feed:
        def next64(self):
            return next(raw)

        def next_double(self):
            return (next(raw) >> 11) * (1.0 / 9007199254740992.0)

    f = Feed()
    got = np.array([tr.standard_exponential(f, ke, we, fe) for _ in range(1_000_000)])
    want = np.random.Generator(np.random.PCG64(2024)).standard_exponential(1_000_000)
    assert np.array_equal(got, want)


def test_round6_matches_python():
    rng = random.Random(5)
    xs = [rng.random() * 10 ** rng.randint(-9, 5) for _ in range(50_000)]
    xs += [0.0, 5e-7, 1.0000005, 0.1234565, 599.9999995, 2.5e-7]
    for x in xs:
        assert tr.round6(x) == round(x, 6), x


@pytest.mark.parametrize("spec", [(24, 1.5, 2.69, 600.0, 3), (10, 1.5, 3.197988, 600.0, 1),
                                  (100, 1.5, 2.38287, 120.0, 16), (5, 0.5, 9.0, 50.0, 0),
                                  (1, 1.0, 0.3, 80.0, 2 ** 33 + 1)])
def test_generator_restatement_equals_gen_zipf(spec):
    n, s, rate, dur, seed = spec
    ke, we, fe = _tables()
    names = list(default_profiles(n))
    rates = zipf_rates(n, s, rate)
    ent = []
    for k in range(n):
        ent += [(t, names[k]) for t in tr.stream(seed, k, rates[k], dur, ke, we, fe)]
    ent.sort(key=lambda e: (e[0], e[1]))
    assert ent == gen_zipf(n, s, rate, dur, seed).entries
