"""CPU, world_size 2 over gloo: the multi-GPU host logic (batch shard split,
filter broadcast, max-over-ranks timing reduction, gather-and-compare).
The per-shard compute here is the CPU oracle (test infrastructure); on GPUs the
same shards go through the C-ABI (bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_06410_b200.shard import batch_slice, max_over_ranks, shard_params, split_range


def test_split_range_matches_reference():  # threads.hpp:20-25
    assert [split_range(10, r, 3) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [split_range(128, r, 8) for r in range(8)] == [(16 * r, 16 * r + 16) for r in range(8)]
    assert [split_range(2, r, 4) for r in range(4)] == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for n in (1, 7, 64, 256):
        for w in (1, 2, 4, 8):
            parts = [split_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restatement
    orc = Restatement()
    cp = dict(k_n=8, k_h=3, k_w=3, c_i=4, h_i=9, w_i=7, b=5, s=1, p=1)
    # filters: only rank 0 has the real values; broadcast replicates them
    g = np.random.default_rng(7)
    F_full = g.uniform(-1, 1, (8, 3, 3, 4)).astype(np.float32)
    F = torch.from_numpy(np.asfortranarray(F_full).reshape(-1, order="F").copy()) if rank == 0 \
        else torch.zeros(8 * 3 * 3 * 4)
    dist.broadcast(F, src=0)
    Fn = np.asfortranarray(F.numpy().reshape((8, 3, 3, 4), order="F"))
    I_full = np.asfortranarray(np.random.default_rng(11).uniform(-1, 1, (9, 7, 4, 5)).astype(np.float32))
    b0, b1, cpl = shard_params(cp, rank, world)
    O_local = orc.conv_gemm(Fn, np.asfortranarray(batch_slice(I_full, b0, b1)), vars(cpl))
    # gather shards on rank 0 (outside any timed region)
    flat = torch.from_numpy(O_local.reshape(-1, order="F").copy())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([flat.numel()]))
    maxn = max(int(s.item()) for s in sizes)
    padded = torch.zeros(maxn)
    padded[: flat.numel()] = flat
    bufs = [torch.zeros(maxn) for _ in range(world)]
    dist.all_gather(bufs, padded)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        O_full = orc.conv_gemm(Fn, I_full, cp)
        parts = [b[: int(s.item())].numpy() for b, s in zip(bufs, sizes)]
        got = np.concatenate(parts)  # batch outermost -> shards concatenate in storage order
        out.put((bool(np.array_equal(got, O_full.reshape(-1, order="F"))), t,
                 bool(np.array_equal(Fn, F_full))))
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    equal, tmax, f_ok = q.get(timeout=10)
    assert f_ok, "filter broadcast did not replicate rank 0's filters"
    assert equal, "concatenated batch shards differ from the full-batch conv"
    assert tmax == 2.0, "max over ranks"


def _product_worker(rank, world, port, out):
    """One rank of a batch-sharded run of THE PRODUCT: its shard through the C-ABI on
    cuda:0 (the driver box has one GPU; the ranks share it but never wait on each other's
    kernels -- there is no collective in the data path), the filters broadcast over gloo,
    the output shards gathered over gloo for the check."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2005_06410_b200 as cg
    torch.cuda.set_device(0)
    cp = dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=28, w_i=28, b=11, s=2, p=1)
    g = np.random.default_rng(17)
    F_full = np.asfortranarray(g.uniform(-1, 1, (128, 3, 3, 64)).astype(np.float32))
    I_full = np.asfortranarray(g.uniform(-1, 1, (28, 28, 64, 11)).astype(np.float32))
    F = torch.from_numpy(np.asfortranarray(F_full).reshape(-1, order="F").copy()) if rank == 0 \
        else torch.zeros(F_full.size)
    dist.broadcast(F, src=0)  # filters replicated once, outside any timed region
    Fn = np.asfortranarray(F.numpy().reshape(F_full.shape, order="F"))
    b0, b1, cpl = shard_params(cp, rank, world)
    out_local = {}
    for prec in ("tf32", "3xtf32"):
        O = cg.conv(Fn, np.asfortranarray(batch_slice(I_full, b0, b1)), vars(cpl), precision=prec)
        flat = torch.from_numpy(O.reshape(-1, order="F").copy())
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([flat.numel()]))
        maxn = max(int(s.item()) for s in sizes)
        padded = torch.zeros(maxn)
        padded[: flat.numel()] = flat
        bufs = [torch.zeros(maxn) for _ in range(world)]
        dist.all_gather(bufs, padded)
        if rank == 0:
            out_local[prec] = np.concatenate([b[: int(s.item())].numpy() for b, s in zip(bufs, sizes)])
    if rank == 0:
        from oracle.oracle import Restatement, per_output_error
        orc = Restatement()
        ref = orc.conv_gemm(F_full, I_full, cp)
        scale = orc.output_scale(F_full, I_full, cp)
        errs = {p: per_output_error(v.reshape(ref.shape, order="F"), ref, scale) for p, v in out_local.items()}
        out.put(errs)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_two_ranks_product_shards():
    """World size 2: each rank runs its split_range shard (threads.hpp:20-25) through the
    B200 operator; the concatenated shards match the oracle's full-batch convolution at
    the north-star bars."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    errs = q.get(timeout=10)
    assert errs["tf32"] <= 5e-3 and errs["3xtf32"] <= 1e-5, errs
