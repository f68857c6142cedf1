"""World-size-2 gloo test of the multi-GPU host path (paper_2407_19871_b200/dist.py):
key broadcast from rank 0, static sharding, per-rank gate evaluation, gather to rank 0.
No GPU: each rank evaluates its shard with the CPU oracle standing in for its GPU, so
this checks the plumbing the NCCL path uses."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_19871_b200 import TfheParams
    from paper_2407_19871_b200.dist import broadcast_keys, gather_to_root, max_over_ranks, shard_range
    from oracle import oracle as O
    p = TfheParams(80)
    keys, bk, ksk = broadcast_keys(p, seed=7, rank=rank)
    # every rank received the same evaluation keys the oracle derives from the seed
    ok = O.TfheKeys(80, 7)
    assert np.array_equal(bk.numpy().view(np.uint32), ok.bk())
    assert np.array_equal(ksk.numpy().view(np.uint32), ok.ksk())
    assert np.array_equal(keys.lwe_key, ok.lwe_key)
    total = 5
    A = np.array([0, 1, 1, 0, 1], np.uint8)
    B = np.array([1, 1, 0, 0, 1], np.uint8)
    a = keys.encrypt_bits(A, 11)   # the client's full batch (same seed on every rank)
    b = keys.encrypt_bits(B, 12)
    lo, hi = shard_range(total, rank, world)
    out = ok.gate_batch("nand", a[lo:hi], b[lo:hi]) if hi > lo else np.zeros((0, p.n + 1), np.uint32)
    full = gather_to_root(torch.from_numpy(out.view(np.int32)), total, rank, world)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        got = keys.decrypt_bits(full.numpy().view(np.uint32))
        np.save(os.path.join(outdir, "got.npy"), got)
        np.save(os.path.join(outdir, "t.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2407_19871_b200.dist import shard_range
    for total in (0, 1, 7, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_two_rank_gloo_sharded_gates(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "got.npy")
    assert list(got) == [1, 0, 1, 1, 0]  # NAND
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0  # max over ranks


def _sharded_worker(rank, world, port, outdir, mode, Q, R, l, m):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from plain_backend import PlainBackend
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.dist import ShardedLocPir
    b = W.make_batch(Q, R, l, m, seed=123)  # same seeded batch on every rank
    for q in range(min(Q, R)):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    be = PlainBackend()
    run = ShardedLocPir(be, b, rank, world, mode, seed=5)
    run.launch()
    got = run.results()
    # XOR units of this rank's programs: the ranks' sum must equal the reference N*m
    xors = 0
    for p in (run.prog, run.combine):
        if p is not None:
            xors += sum(1 for op in p.ops if (op.kind if not isinstance(op, tuple) else op[0]) == 2)
    import torch
    t = torch.tensor([xors], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        np.save(os.path.join(outdir, "got.npy"), got)
        np.save(os.path.join(outdir, "truth.npy"), b.truth())
        np.save(os.path.join(outdir, "xors.npy"), np.array([int(t.item())]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,world,Q,R", [("boxes", 2, 3, 9), ("boxes", 3, 2, 2),
                                            ("queries", 2, 5, 4), ("queries", 3, 2, 3)])
def test_sharded_locpir_gloo(tmp_path, mode, world, Q, R):
    """box-sharded (cfg3: partial roots all-gathered, rank-0 combine level)
    and query-sharded (cfg4/cfg5: outputs gathered to rank 0) LocPIR over gloo, incl. a
    rank with an empty shard; results == plaintext truth and total XOR units == N*m."""
    l, m = 8, 3
    mp.start_processes(_sharded_worker, args=(world, _free_port(), str(tmp_path), mode, Q, R, l, m),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(tmp_path / "got.npy")
    assert np.array_equal(got, np.load(tmp_path / "truth.npy"))
    assert int(np.load(tmp_path / "xors.npy")[0]) == Q * R * m


def test_chunked_query_programs_match_truth():
    """Query batches evaluated as several programs sharing one scratch region (the bench's
    stated-size cfg4/cfg5 runs) give the same answers as one program."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plain_backend import PlainBackend
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.dist import ShardedLocPir
    b = W.make_batch(7, 3, 8, 3, seed=99)
    for q in range(3):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    one = ShardedLocPir(PlainBackend(), b, 0, 1, "queries", seed=5)
    chunked = ShardedLocPir(PlainBackend(), b, 0, 1, "queries", seed=5, chunk=3)
    assert len(chunked.progs) == 3 and len(one.progs) == 1
    assert chunked.lay.total < one.lay.total
    for r in (one, chunked):
        r.launch()
        assert np.array_equal(r.results(), b.truth())
