"""N > 1 host logic on CPU (world size 2, gloo): batch sharding with a zero-padded
all-reduce reproduces the single-process result bitwise; term sharding sums to the
full-Hamiltonian result.  The per-rank compute here is the CPU oracle standing in
for the GPU kernels (no device in this container); the partition rule is the
engine's own: paper_2602_14167_b200.dist.shard_range calls the C-ABI's
qf_shard_range, the function csrc/capi.cpp's sharded evaluation uses.  The same
split through the CUDA engine is replayed on one GPU by
tests/test_gpu_api.py::test_virtual_ranks_batch_and_term_sharding."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from oracle import pyoracle as po
    from paper_2602_14167_b200.dist import shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, ops, P = po.hea_template(6, 2)
    a = po.Ansatz(n, ops, P)
    h = po.random_sum(6, 24, po.Rng(3), True)
    streams = po.Rng(11).split(7)
    th = np.array([[s.normal() for _ in range(P)] for s in streams])
    B = th.shape[0]
    buf = torch.zeros(B * (1 + P), dtype=torch.float64)
    if mode == "batch":
        b0, b1 = shard_range(B, rank, world)
        if b1 > b0:
            E, G = po.energy_grad_batch(a, th[b0:b1], h, mode="adjoint")
            buf[b0:b1] = torch.from_numpy(E)
            buf[B:].view(B, P)[b0:b1] = torch.from_numpy(G)
    else:
        t0, t1 = shard_range(len(h.wr), rank, world)
        hr = po.Hamil(n, h.codes[t0:t1], h.wr[t0:t1] + 1j * h.wi[t0:t1])
        E, G = po.energy_grad_batch(a, th, hr, mode="adjoint")
        buf[:B] = torch.from_numpy(E)
        buf[B:] = torch.from_numpy(G.reshape(-1))
    dist.all_reduce(buf)
    if rank == 0:
        E_full, G_full = po.energy_grad_batch(a, th, h, mode="adjoint")
        out.put((buf[:B].numpy().copy(), buf[B:].view(B, P).numpy().copy(), E_full, G_full))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["batch", "terms"])
def test_world2_sharding(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    E, G, Ef, Gf = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    if mode == "batch":
        assert np.array_equal(E, Ef) and np.array_equal(G, Gf)
    else:
        assert np.abs(E - Ef).max() < 1e-12 and np.abs(G - Gf).max() < 1e-12


def test_shard_range_partitions():
    from paper_2602_14167_b200.dist import shard_range
    for count in (0, 1, 7, 1024, 2000):
        for world in (1, 2, 3, 8):
            rs = [shard_range(count, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == count
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
