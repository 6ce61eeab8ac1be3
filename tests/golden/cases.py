"""Deterministic parity-case generators shared by make_golden.py and tests.

Each case is a JSON-serialisable dict:
  trace:    {"gen": [n, zipf_s, rate, duration, seed], "names": [...]?}
            or {"entries": [[t, name], ...]}
  profiles: {"default": [n, mem_mb?, compute_share?]} or
            {"explicit": [[name, warm, cold, mem, share, weight], ...]}
  policy:   mqfq | fcfs | batch | sjf | fcfs_naive
  sched:    SchedulerConfig kwargs (t_overrun, alpha, default_ttl_s, weights)
  devices:  list of DeviceConfig kwargs
  tau_inc:  run_simulation(tau_includes_overheads=...)
  scripted: {"arrivals", "execs", "d", "deny"} -> oracles.drive() instances

Families:
  appendix_b  default.cfg / medium.cfg x 5 policies
  engine      the reference's test_engine.py scenarios
  fuzz        A1-style random instances over every device/scheduler knob
  c3 / c2 / c4  samples of the BASELINE configs (F=100 sweep grid, F=200
              Azure-shaped, F=512 heterogeneous memory stress)
  a8 / a11    the acceptance suite's scripted oracle instances
              (test_acceptance.py:256-280,324-343), same RNG recipes
"""

from __future__ import annotations

import random

REF_FUNCS = [
    ("isoneural", 0.026, 9.963), ("roberta", 0.268, 15.481), ("fft", 0.897, 3.322),
    ("pathfinder", 1.472, 1.797), ("needle", 1.979, 2.177), ("lud", 2.050, 2.359),
    ("imagenet", 2.253, 11.286), ("ffmpeg", 4.483, 4.612),
]
POLICIES = ["mqfq", "fcfs", "batch", "sjf", "fcfs_naive"]


def _zipf_shares(n, s):
    w = [(k + 1) ** (-s) for k in range(n)]
    tot = sum(w)
    return [x / tot for x in w]


def _rho_rate(warms, s, rho):
    shares = _zipf_shares(len(warms), s)
    mean_exec = sum(sh * w for sh, w in zip(shares, warms))
    return rho * 1.8 / max(mean_exec, 0.05)


def appendix_b():
    out = []
    default = dict(trace={"gen": [24, 1.5, 2.69, 600.0, 1]}, profiles={"default": [24]},
                   sched={"t_overrun": 10.0, "alpha": 2.0},
                   devices=[{"mem_capacity_mb": 16384.0, "d_max": 2, "pool_max_containers": 32}])
    medium = dict(trace={"gen": [19, 1.5, 2.0, 1500.0, 7]},
                  profiles={"default": [19, 1500.0, 0.46]},
                  sched={"t_overrun": 10.0, "alpha": 2.0},
                  devices=[{"mem_capacity_mb": 16384.0, "d_max": 2, "util_threshold": 0.97,
                            "util_window_s": 0.4, "pcie_mb_per_s": 3000.0,
                            "pool_max_containers": 32}])
    for tag, base in (("default", default), ("medium", medium)):
        for pol in POLICIES:
            c = {k: (v if not isinstance(v, list) else [dict(x) for x in v])
                 for k, v in base.items()}
            c["name"] = f"appendix_b/{tag}/{pol}"
            c["policy"] = pol
            if pol == "fcfs_naive":
                c["devices"] = [dict(d, pool_enabled=False) for d in c["devices"]]
            out.append(c)
    return out


def engine_cases():
    f14 = [["f", 1.0, 4.0, 100.0, 0.4, 1.0]]
    f12 = [["f", 1.0, 2.0, 100.0, 0.4, 1.0]]
    ff = [["f", 1.0, 1.0, 100.0, 0.9, 1.0]]
    return [
        dict(name="engine/empty", trace={"entries": []}, profiles={"default": [4]}),
        dict(name="engine/single_cold", trace={"entries": [[2.0, "f"]]},
             profiles={"explicit": f14}),
        dict(name="engine/same_time", trace={"entries": [[1.0, "fft"], [1.0, "roberta"]]},
             profiles={"default": [4]}),
        dict(name="engine/monitor_tail", trace={"entries": [[0.0, "fft"]]},
             profiles={"default": [4]}),
        dict(name="engine/cascade", trace={"entries": [[0.0, "f"], [0.0, "f"]]},
             profiles={"explicit": ff}, devices=[{"d_max": 1}]),
        dict(name="engine/alpha0_swap", trace={"entries": [[0.0, "f"], [10.0, "f"]]},
             profiles={"explicit": f12}, sched={"alpha": 0.0}),
        dict(name="engine/anticipation", trace={"entries": [[0.0, "f"], [3.5, "f"]]},
             profiles={"explicit": f12}, sched={"alpha": 2.0, "default_ttl_s": 2.0}),
        dict(name="engine/expired_swap", trace={"entries": [[0.0, "f"], [30.0, "f"]]},
             profiles={"explicit": f12}, sched={"alpha": 2.0, "default_ttl_s": 2.0}),
        dict(name="engine/conservation", trace={"gen": [4, 1.5, 1.0, 60.0, 3]},
             profiles={"default": [4]}),
        dict(name="engine/clock", trace={"gen": [3, 1.2, 1.0, 30.0, 1]},
             profiles={"default": [3]}),
        dict(name="engine/determinism", trace={"gen": [5, 1.5, 1.5, 90.0, 11]},
             profiles={"default": [5]}),
        dict(name="engine/multi_device", trace={"gen": [6, 1.5, 2.5, 60.0, 13]},
             profiles={"default": [6]}, devices=[{}, {}]),
        dict(name="engine/littles_law_lite", trace={"gen": [1, 1.5, 0.8, 400.0, 1]},
             profiles={"explicit": [["isoneural", 0.897, 3.322, 1500.0, 0.4, 1.0]]}),
    ]


def fuzz_case(trial: int) -> dict:
    rng = random.Random(7_000_000 + trial)
    n = rng.randint(1, 12)
    s = rng.choice([0.8, 1.2, 1.5])
    hetero = rng.random() < 0.6
    rows = []
    for i in range(n):
        base, warm, cold = REF_FUNCS[i % 8]
        name = base if i < 8 else f"{base}_c{i // 8}"
        if hetero:
            mem = rng.choice([256.0, 512.0, 1024.0, 1500.0, 3000.0, 6000.0, 1234.5])
            share = rng.choice([0.1, 0.38, 0.46, 0.7, 0.95, 0.333])
            weight = rng.choice([1.0, 1.0, 2.0, 0.5, 3.0])
        else:
            mem, share, weight = 1500.0, 0.38, 1.0
        rows.append([name, warm, cold, mem, share, weight])
    max_mem = max(r[3] for r in rows)
    ndev = rng.choice([1, 1, 1, 2, 2, 3])
    devices = []
    for _ in range(ndev):
        d = {
            "mem_capacity_mb": max(max_mem, rng.choice([4000.0, 6000.0, 8000.0, 16384.0])),
            "d_max": rng.randint(1, 4),
            "util_threshold": rng.choice([0.9, 0.97, 0.75, 1.0, 0.6]),
            "pcie_mb_per_s": rng.choice([12000.0, 3000.0, 700.0]),
            "interference_beta": rng.choice([0.1, 0.0, 0.3]),
            "monitor_period_s": rng.choice([0.2, 0.2, 0.1, 0.25]),
            "util_window_s": rng.choice([1.0, 0.4, 2.0]),
            "pool_max_containers": rng.choice([1, 2, 4, 8, 32]),
            "pool_enabled": rng.random() < 0.9,
            "dynamic_d": rng.random() < 0.3,
            "prefetch_overlap_s": rng.choice([0.0, 0.0, 0.05, 0.5]),
        }
        devices.append(d)
    policy = rng.choice(POLICIES + ["mqfq", "mqfq", "mqfq"])
    if policy == "fcfs_naive":
        for d in devices:
            d["pool_enabled"] = False
    sched = {"t_overrun": rng.choice([0.0, 1.0, 5.0, 10.0, 0.5]),
             "alpha": rng.choice([0.0, 0.5, 1.0, 2.0, 4.0]),
             "default_ttl_s": rng.choice([2.0, 0.5, 5.0])}
    if rng.random() < 0.2:
        sched["weights"] = {rows[k][0]: rng.choice([0.5, 2.0, 4.0])
                            for k in range(n) if rng.random() < 0.5}
    rho = rng.uniform(0.5, 1.4)
    rate = _rho_rate([r[1] for r in rows], s, rho)
    dur = rng.uniform(20.0, 150.0)
    return dict(name=f"fuzz/{trial}", trace={"gen": [n, s, rate, dur, trial + 1],
                                           "names": [r[0] for r in rows]},
                profiles={"explicit": rows}, policy=policy, sched=sched, devices=devices,
                tau_inc=rng.random() < 0.2)


def c3_case(idx: int) -> dict:
    """One point of the C3 grid: F=100, s=1.5, rho=1."""
    Ts = [0.0, 1.0, 2.0, 5.0, 10.0, 20.0, 50.0, 100.0]
    As = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 8.0]
    Ds = [1, 2, 3, 4]
    seed = idx % 16 + 1
    rest = idx // 16
    d = Ds[rest % 4]
    a = As[(rest // 4) % 8]
    t = Ts[(rest // 32) % 8]
    return dict(name=f"c3/{idx}", trace={"gen": [100, 1.5, 2.382870, 600.0, seed]},
                profiles={"default": [100]}, policy="mqfq",
                sched={"t_overrun": t, "alpha": a}, devices=[{"d_max": d}])


def c2_case(idx: int) -> dict:
    rates = [1.12, 1.69, 1.94, 4.26, 2.69, 2.57, 2.55, 1.79, 1.12]
    pol = ["mqfq", "fcfs", "batch"][idx % 3]
    r = rates[(idx // 3) % 9]
    seed = idx // 27 + 1
    return dict(name=f"c2/{idx}", trace={"gen": [200, 1.5, r, 600.0, seed]},
                profiles={"default": [200]}, policy=pol, devices=[{}])


def c4_case(idx: int) -> dict:
    """Large-flow stress (BASELINE C4, shortened): heterogeneous mem by rank."""
    n = 512
    rows = []
    mems = [256.0, 512.0, 1024.0, 1500.0, 3000.0]
    for i in range(n):
        base, warm, cold = REF_FUNCS[i % 8]
        name = base if i < 8 else f"{base}_c{i // 8}"
        rows.append([name, warm, cold, mems[i % 5], 0.38, 1.0])
    pool = [32, 256][idx % 2]
    return dict(name=f"c4/{idx}", trace={"gen": [n, 0.5, 2.0, 300.0, idx + 1],
                                        "names": [r[0] for r in rows]},
                profiles={"explicit": rows}, policy=["mqfq", "fcfs"][idx // 2 % 2],
                devices=[{"d_max": 4, "pool_max_containers": pool}])


def a8_case(trial: int) -> dict:
    """test_acceptance.py:256-280, same RNG draws in the same order."""
    rng = random.Random(10_000 + trial)
    n = rng.randint(2, 4)
    names = [f"f{i}" for i in range(n)]
    arrivals = sorted((round(rng.uniform(0, 30), 3), rng.choice(names))
                      for _ in range(rng.randint(4, 20)))
    execs = [round(rng.uniform(0.1, 5.0), 3) for _ in range(60)]
    d = rng.choice([1, 2, 3])
    deny = rng.choice([0, 0, 3, 5])
    t_overrun = rng.choice([0.0, 1.0, 5.0, 10.0])
    alpha = rng.choice([0.0, 1.0, 2.0])
    return dict(name=f"a8/{trial}", policy="mqfq",
                sched={"t_overrun": t_overrun, "alpha": alpha},
                scripted={"arrivals": [list(a) for a in arrivals], "execs": execs,
                          "d": d, "deny": deny, "names": names})


def a11_case(trial: int) -> dict:
    """test_acceptance.py:324-343 (T=0, D=1, alpha=0)."""
    rng = random.Random(20_000 + trial)
    n = rng.randint(2, 5)
    names = [f"f{i}" for i in range(n)]
    arrivals = sorted((round(rng.uniform(0, 40), 3), rng.choice(names))
                      for _ in range(rng.randint(5, 25)))
    execs = [round(rng.uniform(0.1, 4.0), 3) for _ in range(80)]
    return dict(name=f"a11/{trial}", policy="mqfq",
                sched={"t_overrun": 0.0, "alpha": 0.0},
                scripted={"arrivals": [list(a) for a in arrivals], "execs": execs,
                          "d": 1, "deny": 0, "names": names})


C4_MEM_MB = [256.0, 512.0, 1024.0, 1500.0, 3000.0]


def c1_cases() -> list:
    """BASELINE C1's 10-function variant of configs/default.cfg (rate
    3.197988, 600 s, seed 1 -> 1,875 arrivals), under every
    policy.  default.cfg itself is appendix_b's default/* family."""
    out = []
    for pol in POLICIES:
        out.append(dict(name=f"c1/f10_{pol}", trace={"gen": [10, 1.5, 3.197988, 600.0, 1]},
                        profiles={"default": [10]}, policy=pol,
                        sched={"t_overrun": 10.0, "alpha": 2.0},
                        devices=[{"mem_capacity_mb": 16384.0, "d_max": 2,
                                  "pool_max_containers": 32}]))
    return out


def c4x_case(idx: int) -> dict:
    """BASELINE C4 at its full flow count (the bench's sweep.c4 profiles:
    4096 default-profile functions, mem_mb by rank mod 5, share 0.38; Zipf
    0.5 at 2 rps; 16 GB device, D=4, pool 32 / 256) on short traces, so the
    reference finishes in seconds to minutes; c4x/6-7 are two of the bench's
    own 1800 s C4 simulations (seeds 1 and 2)."""
    dur, pol, pool, seed = [(60.0, "mqfq", 32, 101), (60.0, "mqfq", 256, 102),
                            (60.0, "fcfs", 32, 103), (300.0, "mqfq", 32, 104),
                            (300.0, "mqfq", 256, 105), (300.0, "fcfs", 256, 106),
                            (1800.0, "mqfq", 32, 1), (1800.0, "fcfs", 256, 2)][idx]
    return dict(name=f"c4x/{idx}", trace={"gen": [4096, 0.5, 2.0, dur, seed]},
                profiles={"c4": [4096]}, policy=pol,
                devices=[{"d_max": 4, "pool_max_containers": pool}])


def extra_cases() -> list:
    """Round-2 families, kept out of all_cases(): c4x's 4096-flow layout would
    change the build the 1560-case batch runs in.  Golden file:
    reference_golden_extra.json (make_golden.py --extra)."""
    return c1_cases() + [c4x_case(i) for i in range(8)]


def all_cases(n_fuzz=400, n_c3=24, n_c2=9, n_c4=4, n_a8=1000, n_a11=100):
    cases = appendix_b() + engine_cases()
    cases += [fuzz_case(i) for i in range(n_fuzz)]
    cases += [c3_case(i * 173 % 4096) for i in range(n_c3)]
    cases += [c2_case(i * 37 % 12312) for i in range(n_c2)]
    cases += [c4_case(i) for i in range(n_c4)]
    cases += [a8_case(i) for i in range(n_a8)]
    cases += [a11_case(i) for i in range(n_a11)]
    return cases
