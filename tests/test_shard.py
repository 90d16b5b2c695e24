"""CPU multi-process tests (gloo, world size 2) of the frame sharding + detection gather
used by bench.py --gpus N.  Each rank runs the receiver on its frame shard (the CPU
oracle stands in for the GPU kernels here) and rank 0 must end up with exactly the
single-process detections, in frame order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_03883_b200.shard import DetectionGather, pack, shard_range, unpack


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for frames in (1, 7, 8192, 8193):
        for world in (1, 2, 3, 8):
            rs = [shard_range(frames, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == frames
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_c_abi_shard_range_matches():
    # the C-ABI's multi-device sharding (ofdmr_shard_range) is the same partition as shard.py's
    import ctypes as C

    from paper_2209_03883_b200 import _native

    lib = _native.lib()
    for frames in (1, 7, 8192, 8193, 10**9 + 7):
        for world in (1, 2, 3, 8):
            for r in range(world):
                lo, hi = C.c_int64(), C.c_int64()
                lib.ofdmr_shard_range(frames, r, world, C.byref(lo), C.byref(hi))
                assert (lo.value, hi.value) == shard_range(frames, r, world)


def test_pack_roundtrip():
    d = torch.randint(0, 1024, (5, 8), dtype=torch.int32)
    v = torch.randint(-128, 128, (5, 8), dtype=torch.int32)
    p = torch.rand(5, 8, dtype=torch.float32)
    c = torch.randint(0, 9, (5,), dtype=torch.int32)
    d2, v2, p2, c2 = unpack(pack(d, v, p, c), 8)
    assert torch.equal(d, d2) and torch.equal(v, v2) and torch.equal(p, p2) and torch.equal(c, c2)


def _oracle_dets(frames, first, count, k):
    import oracle as O
    from paper_2209_03883_b200 import configs, gen

    cfg = configs.CFG4.replace(n=128, m=32, n_prime=128, m_prime=32, n_cp=16, max_targets=k, range_hi=40.0)
    fb = gen.frames(cfg, first, count, threads=1)
    rc = O.rx_config(cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.estimator, cfg.n_cp, cfg.window, cfg.pfa)
    d, v, w, cnt, _, _ = O.receive_batch(rc, fb.y, fb.x, fb.sigma2, k, fb.n_targets, threads=1)
    return (torch.from_numpy(d.astype(np.int32)), torch.from_numpy(v.astype(np.int32)),
            torch.from_numpy(w.astype(np.float32)), torch.from_numpy(cnt.astype(np.int32)))


def _worker(rank, world, port, frames, k, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(frames, rank, world)
    d, v, w, c = _oracle_dets(frames, lo, hi - lo, k)
    g = DetectionGather(frames, k, rank, world, torch.device("cpu"))
    full = g(d, v, w, c)
    if rank == 0:
        torch.save(full, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("frames", [6, 7])
def test_gloo_world2_gather_matches_single_process(tmp_path, frames):
    k = 8
    out = str(tmp_path / "full.pt")
    mp.start_processes(_worker, args=(2, _free_port(), frames, k, out), nprocs=2, join=True, start_method="spawn")
    full = torch.load(out)
    ref = pack(*_oracle_dets(frames, 0, frames, k))
    assert full.shape == ref.shape
    assert torch.equal(full, ref)
