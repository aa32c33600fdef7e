"""Row sharding + all-gather host logic, world size 2 over gloo on CPU; the
per-rank compute is the CPU oracle injected by the test (the product path
uses the CUDA engine, covered on the GPU by tests/test_gemv_gpu.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_10467_b200 import MultiPrecisionModel, QuantConfig, ScaleTensor
from paper_2510_10467_b200.model import BitPlaneSet
from paper_2510_10467_b200.parallel import row_shard_bounds, shard_model


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _model(rows, cols, asym, seed):
    from oracle import anybcq_oracle as O
    words = O.random_words(3, rows, cols, seed)
    rng = np.random.default_rng(seed)
    G = -(-cols // 128)
    sets = {p: ScaleTensor(rng.random((p, rows, G)).astype(np.float32),
                           rng.standard_normal((rows, G)).astype(np.float32) if asym else None, 128)
            for p in (2, 3)}
    return MultiPrecisionModel(BitPlaneSet(3, rows, cols, words), sets, 2, 3,
                               QuantConfig(128, "asymmetric" if asym else "symmetric", 0))


def test_row_shard_bounds_cover_rows():
    for rows in (1, 15, 16, 17, 100, 4096, 14336):
        for world in (1, 2, 3, 4, 8):
            spans = [row_shard_bounds(rows, world, r) for r in range(world)]
            flat = [i for lo, hi in spans for i in range(lo, hi)]
            assert flat == list(range(rows))
            assert all(lo % 16 == 0 or lo == rows for lo, _ in spans)


def test_shard_model_matches_rows():
    from oracle import anybcq_oracle as O
    m = _model(50, 300, True, 1)
    x = O.random_gaussian(1, 300, 2).ravel()
    full = O.gemv_lut(m.bitplanes.words, 300, 128, m.scale_sets[3].alpha, m.scale_sets[3].offset, 3, x)
    sh = shard_model(m, 16, 48)
    part = O.gemv_lut(sh.bitplanes.words, 300, 128, sh.scale_sets[3].alpha, sh.scale_sets[3].offset, 3, x)
    assert np.array_equal(part, full[16:48])


def _worker(rank, world, port, rows, cols, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import anybcq_oracle as O
        from paper_2510_10467_b200.parallel import RowShardedGemv

        m = _model(rows, cols, rank >= 0, 7)

        def local(p, xt, eng=None):
            sh = eng.shard
            y = O.gemv_lut(sh.bitplanes.words, cols, 128, sh.scale_sets[p].alpha,
                           sh.scale_sets[p].offset, p, xt.numpy())
            return torch.from_numpy(y.astype(np.float32))

        eng = RowShardedGemv(m, local_gemv=lambda p, xt: local(p, xt, eng), dtype=torch.float32)
        x = torch.from_numpy(O.random_gaussian(1, cols, 3).ravel())
        y = eng.gemv(2, x).clone()
        assert eng.gemv(2, x).data_ptr() == eng.y.data_ptr()   # preallocated: y is the gather buffer
        want = O.gemv_lut(m.bitplanes.words, cols, 128, m.scale_sets[2].alpha, m.scale_sets[2].offset, 2, x.numpy())
        q.put((rank, float(np.max(np.abs(y.numpy() - want.astype(np.float32)))), tuple(y.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows", [64, 50])
def test_row_sharded_gemv_allgather_gloo(rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, 256, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, shape in res:
        assert shape == (rows,) and err == 0.0, (rank, err)
