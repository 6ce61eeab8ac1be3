"""CPU tests of the host side: trace generation fidelity, packing (name
order, validation errors), the sweep builders and their shards."""

from __future__ import annotations

import numpy as np
import pytest

from cases import all_cases
from fingerprint import fp
from golden_check import golden

from paper_2507_08954_b200 import sweep
from paper_2507_08954_b200.core import FunctionProfile
from paper_2507_08954_b200.dist import hist_bin, shard_bounds
from paper_2507_08954_b200.pack import flow_table, pack_trace
from paper_2507_08954_b200.workload import default_profiles, gen_zipf


@pytest.mark.parametrize("name", ["appendix_b/default/mqfq", "appendix_b/medium/mqfq",
                                  "c3/0", "c2/0", "c4/0"])
def test_trace_generation_matches_reference(name):
    """gen_zipf reproduces the reference's trace bits (workload.py:82-111)."""
    case = {c["name"]: c for c in all_cases(n_fuzz=0, n_a8=0, n_a11=0)}[name]
    n, s, rate, dur, seed = case["trace"]["gen"][:5]
    prof = case.get("profiles", {"default": [8]})
    names = case["trace"].get("names") or list(default_profiles(*prof["default"]))[:n]
    tr = gen_zipf(n, s, rate, dur, seed, names=names)
    assert fp([(t, nm) for t, nm in tr.entries]) == golden()[name]["fp"]["trace"]


def test_pack_ranks_by_python_string_order():
    ents = [(0.0, "fft"), (0.5, "ffmpeg"), (1.0, "fft_c1"), (1.0, "fft")]
    pt = pack_trace(ents)
    assert pt.names == ["ffmpeg", "fft", "fft_c1"]          # 'ffmpeg' < 'fft' in str order
    assert pt.flow.tolist() == [1, 0, 2, 1]
    assert pt.arrival.dtype == np.float64


def test_pack_validation_mirrors_simulation_init():
    profs = default_profiles(2)
    with pytest.raises(ValueError, match="unknown functions"):
        pack_trace([(0.0, "nope")], profs)
    with pytest.raises(ValueError, match="non-decreasing"):
        pack_trace([(1.0, "isoneural"), (0.5, "isoneural")], profs)


def test_flow_table_weight_override():
    profs = {"a": FunctionProfile("a", 1.0, 2.0, 100.0, 0.4, 3.0),
             "b": FunctionProfile("b", 1.0, 2.0, 100.0, 0.4, 1.0)}
    tab = flow_table(["a", "b"], profs, {"b": 0.5})
    assert tab.weight.tolist() == [3.0, 0.5]                 # weight_of, mqfq.py:88-92


def test_c3_grid_and_shards():
    w = sweep.c3(n_seeds=2, duration=30.0)
    assert len(w.sims) == 8 * 8 * 4 * 2
    ts = sorted({s.t_overrun for s in w.sims})
    assert ts == sweep.C3_T
    assert sorted({s.alpha for s in w.sims}) == sweep.C3_ALPHA
    assert {w.dcfgs[s.device_cfg].d_max for s in w.sims} == {1, 2, 3, 4}
    assert max(s.group for s in w.sims) == 63
    w1 = sweep.build("c3", rank=1, n_seeds=2)
    assert w1.describe["seeds"] == [3, 4]                    # disjoint seed block per rank


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            blocks = [shard_bounds(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))


def test_hist_bin_edges():
    b = hist_bin([0.0, 1e-3, 0.01, 1.0, 1e5, 1e9], 1e-2, 1e5, 64)
    assert b[0] == 0 and b[1] == 0 and b[2] == 0 and b[-1] == 63 and b[-2] == 63
    assert 0 < b[3] < 63


def test_capacity_retry_policy_without_a_gpu(monkeypatch):
    """engine._run_one (run_simulation / Simulation): the engine's own capacity
    statuses are re-run with larger buffers; anything else raises at once."""
    import numpy as np
    from paper_2507_08954_b200 import _abi, engine
    from paper_2507_08954_b200._lib import EngineError

    class FakeEngine:
        def __init__(self, statuses):
            self.statuses, self.calls = list(statuses), []

        def prepare(self, sims, outputs, early_exit, **kw):
            self.calls.append((int(sims[0].max_events), dict(kw)))

        def launch(self):
            pass

        def synchronize(self):
            self.st = self.statuses.pop(0)
            if self.st:
                raise EngineError("simulation 0 failed")

        def output(self, oid):
            return np.array([self.st], dtype=np.int32)

        def batch_info(self):
            return {"event_capacity": 352}                 # the auto capacity that overflowed

    sim = _abi.Sim()
    eng = FakeEngine([1, 3, 5, 0])
    monkeypatch.setattr(engine, "BatchResult", lambda e: "ok")   # no device outputs here
    assert engine._run_one(eng, sim, 100, _abi.WANT_STATS, True, audit_util_cap=8) == "ok"
    (m0, k0), (m1, k1), (m2, k2), (m3, k3) = eng.calls
    assert k1["event_capacity"] == 4 * 352                # event-pool overflow: 4x what overflowed
    assert m2 == 16 * 64 * (100 + 1024)                   # watchdog: 16x the event budget
    assert k3["audit_util_cap"] == 32 and k3["event_log_cap"] == 4 << 16   # output overflow
    bad = FakeEngine([4])                                  # past event: the reference's error
    with pytest.raises(EngineError):
        engine._run_one(bad, sim, 100, _abi.WANT_STATS, True)
