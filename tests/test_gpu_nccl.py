"""The C-ABI NCCL collective (gfq_reduce_nccl, dlopen'd libnccl) on one GPU:
a single-rank communicator made through gfq_nccl_comm_init must leave the
summed histograms unchanged and gather exactly this rank's summary rows.
(Multi-rank sharding and reduction are covered on CPU by test_dist_gloo.)"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_single_rank_reduce_nccl():
    import torch
    from paper_2507_08954_b200 import _abi, sweep
    from paper_2507_08954_b200.engine import Engine, NcclComm
    torch.cuda.set_device(0)
    eng = Engine(0)
    w = sweep.build("c3", 0, engine=eng, n_seeds=2)
    w.upload(eng)
    eng.prepare(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_HIST, early_exit=True,
                hist_groups=w.groups, hist_rows=w.hist_rows, hist_bins=sweep.HIST_BINS,
                hist_lo_s=sweep.HIST_LO_S, hist_hi_s=sweep.HIST_HI_S)
    eng.launch()
    eng.synchronize()
    hist0 = eng.output(_abi.OUT_HIST).copy()
    summ0 = eng.output(_abi.OUT_SUMMARY).copy()
    comm = NcclComm(1, 0, NcclComm.unique_id())
    out = torch.zeros(summ0.shape[0], dtype=torch.float64, device="cuda")
    eng.launch()
    eng.reduce_nccl(comm, out)
    eng.synchronize()
    torch.cuda.synchronize()
    assert np.array_equal(eng.output(_abi.OUT_HIST), hist0)
    assert np.array_equal(out.cpu().numpy(), summ0)
    comm.close()
    eng.close()
