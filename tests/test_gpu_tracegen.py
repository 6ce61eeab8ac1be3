"""GPU trace generator (gfq_generate_traces, csrc/tracegen.cuh) against the
reference's gen_zipf (workload.py:82-111, numpy 2.3): every generated trace
must equal pack_trace(gen_zipf(...)) bit for bit -- arrival times, flow ids
and touched-name sets -- over the BASELINE sweep shapes and edge cases
(seed 0 and >= 2^32, one function, empty traces, 4096 functions), and
simulating a generated trace must give the same results as the host one."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPECS = ([(100, 1.5, 2.382870, 600.0, s) for s in range(1, 33)] +            # C3
         [(200, 1.5, r, 600.0, s) for r in (1.12, 4.26) for s in (1, 2, 3)] +  # C2
         [(24, 1.5, 2.69, 600.0, 1), (19, 1.5, 2.0, 1500.0, 7),              # Appendix B
          (1, 1.0, 0.5, 100.0, 0), (3, 2.0, 0.01, 5.0, 9),                   # tiny / empty
          (6, 1.5, 1.0, 0.0, 7), (12, 0.8, 30.0, 60.0, 2 ** 33 + 11),        # zero duration, big seed
          (4096, 0.5, 2.0, 1800.0, 1)])                                       # C4


@pytest.fixture(scope="module")
def engine():
    from paper_2507_08954_b200.engine import Engine
    e = Engine(0)
    yield e
    e.close()


def test_generated_traces_equal_gen_zipf(engine):
    from paper_2507_08954_b200.pack import pack_trace
    from paper_2507_08954_b200.workload import gen_zipf
    got = engine.generate_traces(SPECS)
    bad = []
    for spec, g in zip(SPECS, got):
        ref = pack_trace(gen_zipf(*spec).entries)
        if not (g.names == ref.names and np.array_equal(g.arrival, ref.arrival)
                and np.array_equal(g.flow, ref.flow)):
            bad.append(spec)
    assert not bad, bad


def test_many_traces_stress(engine):
    """2000 traces x 100 functions (~2.7M arrivals, the ziggurat rejection
    path ~3x10^4 times) vs numpy."""
    from paper_2507_08954_b200.pack import pack_trace
    from paper_2507_08954_b200.workload import gen_zipf
    specs = [(100, 1.5, 2.38287 * (0.7 + 0.4 * (s % 5) / 4), 600.0, 1000 + s) for s in range(2000)]
    got = engine.generate_traces(specs)
    rng = np.random.default_rng(0)
    check = sorted(rng.choice(len(specs), 200, replace=False).tolist())
    for i in check:
        ref = pack_trace(gen_zipf(*specs[i]).entries)
        assert got[i].names == ref.names and np.array_equal(got[i].arrival, ref.arrival) \
            and np.array_equal(got[i].flow, ref.flow), specs[i]


def test_simulating_generated_traces(engine):
    """A sweep on GPU-generated traces gives the host-generated sweep's
    results (same dispatch counts and statistics)."""
    from paper_2507_08954_b200 import _abi, sweep
    w = sweep.c3(n_seeds=2)
    w.upload(engine)
    a = engine.run(w.sims_array(), outputs=_abi.WANT_STATS)
    ca = engine.output(_abi.OUT_COUNTERS).copy(); sa = engine.output(_abi.OUT_SUMMARY).copy()
    gen = engine.generate_traces([(100, 1.5, sweep.C3_RATE, 600.0, s) for s in (1, 2)])
    for g, t in zip(gen, w.traces):
        assert g.names == t.names
    engine.upload_flowtabs(w.tabs)
    engine.upload_device_cfgs(w.dcfgs)
    engine.run(w.sims_array(), outputs=_abi.WANT_STATS)
    assert np.array_equal(engine.output(_abi.OUT_COUNTERS), ca)
    assert np.array_equal(engine.output(_abi.OUT_SUMMARY), sa)


def test_generate_validation(engine):
    from paper_2507_08954_b200._lib import EngineError
    with pytest.raises(ValueError):
        engine.generate_traces([(0, 1.5, 1.0, 10.0, 1)])
    with pytest.raises(ValueError):
        engine.generate_traces([(4, 1.5, -1.0, 10.0, 1)])
    with pytest.raises(ValueError):
        engine.generate_traces([(4, 0.0, 1.0, 10.0, 1)])
    with pytest.raises(ValueError):
        engine.generate_traces([(4, 1.5, 1.0, 10.0, 1, ["a", "b"])])
    assert engine.generate_traces([(4, 1.5, 1.0, -5.0, 1)])[0].n == 0    # as gen_zipf
    with pytest.raises((ValueError, EngineError)):
        engine.generate_traces([(4, 1.5, 1.0, float("inf"), 1)])
