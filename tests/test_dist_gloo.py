"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in paper_2304_09049_b200/shard.py:
batch sharding of the conv workloads, the output-channel split + row all-gather of config 5,
and the max-over-ranks timing reduction.  The per-rank compute is the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2304_09049_b200 import netrun, shard
        # --- config 5 style: output-channel split + row all-gather
        n = 48
        wl, al = synth.learned_levels(5, 0, synth.T_LEVELS)
        T = oracle.build_lut16(wl, al)
        r0, r1 = shard.row_shard(rank, world, n)
        W = synth.counter_codes(r0 * n, (r1 - r0) * n, (5, n, synth.T_W), "uniform").view(r1 - r0, n).numpy()
        A = synth.counter_codes(0, n * n, (5, n, synth.T_A), "uniform").view(n, n).numpy()
        C_loc = torch.from_numpy(oracle.lut_gemm(W, np.ascontiguousarray(A.T), T))
        C = shard.gather_rows(C_loc, world).numpy()
        # --- conv style: batch shard, per-rank regeneration (no collective), gathered for checking
        L = synth.resnet50_layers()[1]
        imgs = shard.batch_shard(rank, world, 2)
        x = netrun.input_codes(3, 1, L, list(imgs), "cpu").numpy()
        w = netrun.weight_codes(3, 1, L, "cpu").numpy()
        small = type(L)(L.name, 8, 8, 3, 1, 1, 6)  # same generator keys, small shape
        xs = netrun.input_codes(3, 1, small, list(imgs), "cpu").numpy()
        ws_ = netrun.weight_codes(3, 1, small, "cpu").numpy()
        out = torch.from_numpy(oracle.conv2d_direct(xs, ws_, oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM), 1, 1).copy())
        out_all = shard.gather_rows(out, world).numpy()
        t = shard.max_over_ranks(float(rank + 1), world)
        q.put((rank, C, out_all, t, x.shape))
    finally:
        dist.destroy_process_group()


def test_world2_sharding_equals_single_process():
    import oracle
    import synth
    from paper_2304_09049_b200 import netrun
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # single-process references
    n = 48
    wl, al = synth.learned_levels(5, 0, synth.T_LEVELS)
    W = synth.counter_codes(0, n * n, (5, n, synth.T_W), "uniform").view(n, n).numpy()
    A = synth.counter_codes(0, n * n, (5, n, synth.T_A), "uniform").view(n, n).numpy()
    C_ref = oracle.lut_gemm(W, np.ascontiguousarray(A.T), oracle.build_lut16(wl, al))
    L = synth.resnet50_layers()[1]
    small = type(L)(L.name, 8, 8, 3, 1, 1, 6)
    xs = netrun.input_codes(3, 1, small, list(range(4)), "cpu").numpy()
    ws_ = netrun.weight_codes(3, 1, small, "cpu").numpy()
    out_ref = oracle.conv2d_direct(xs, ws_, oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM), 1, 1)
    for rank, C, out_all, t, xshape in res:
        assert np.array_equal(C, C_ref)                 # gathered rows == unsharded GEMM
        assert np.array_equal(out_all, out_ref)         # shards regenerate exactly their images
        assert t == float(world)                        # max over ranks
        assert xshape == (2, L.h, L.h, L.cin)


def test_shard_arithmetic():
    from paper_2304_09049_b200 import shard
    assert list(shard.batch_shard(3, 8, 32)) == list(range(96, 128))
    assert shard.row_shard(7, 8, 16384) == (14336, 16384)
    with pytest.raises(ValueError):
        shard.row_shard(0, 3, 16)
