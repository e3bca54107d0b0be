"""The C-ABI multi-GPU band executor (csrc_gpu_band_exec_*) on the one GPU of
the test box: a one-rank NCCL communicator, both band forms, products equal the
oracle, the async-error poll is clean. The exchange itself needs two or more
GPUs (NCCL refuses two ranks on one device); its lists are pinned on CPU
against the Python plans (tests/test_dist.py)."""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Oracle

import paper_1003_0952_b200 as P

from .helpers import rel_l2

pytestmark = pytest.mark.gpu
O = Oracle()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("form", ["windowed", "gather"])
@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_band_executor_one_rank(group, form, cfg):
    import torch
    from paper_1003_0952_b200.dist import NcclBandSpmv
    a, x, _ = P.config_matrix(cfg)
    ex = NcclBandSpmv(a, form=form)
    L = ex.lists
    assert (L.row_begin, L.row_end, L.n_sends, L.n_recvs) == (0, a.n, 0, 0)
    xd = torch.from_numpy(x[L.x_lo:L.x_hi].copy()).cuda()
    yd = torch.full((L.row_end - L.y_lo,), float("nan"), dtype=torch.float64, device="cuda")
    for refresh in (False, True):
        ex.apply_device(xd, yd, refresh_x=refresh)
        torch.cuda.synchronize()
        assert rel_l2(yd[L.row_begin - L.y_lo:].cpu().numpy(), O.spmv_csrc(a, x)) <= 1e-12
    ex.check()
    ex.close()
