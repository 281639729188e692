"""Host-side multi-process logic of the sharded engine, on CPU with gloo (world size 2).

Covers what runs on the host around the NCCL data path: the generator-word and shot-word
partitions, the ncclUniqueId hand-over, max-over-ranks timing and the assembly of per-rank
tableau columns into the full reference-layout tableau (paper_2603_14641_b200/dist.py).
The device side of the protocol is parity-tested on the GPU (tests/test_gpu_sharded.py).
"""
import os
import socket

import numpy as np
import pytest


def test_shard_range_partitions_generator_words(q):
    for n in [64, 65, 100, 1000, 20000, 180000]:
        k = (n + 63) // 64
        for world in range(1, min(k, 9) + 1):
            ranges = [q.shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0
            for (a0, ak), (b0, _) in zip(ranges, ranges[1:]):
                assert a0 + ak == b0
            assert ranges[-1][0] + ranges[-1][1] == k
            assert min(kg for _, kg in ranges) >= 1
            assert max(kg for _, kg in ranges) - min(kg for _, kg in ranges) <= 1
    with pytest.raises(q.InvalidArgument):
        q.shard_range(100, 3, 0)  # k = 2
    with pytest.raises(q.InvalidArgument):
        q.shard_range(1000, 2, 2)


def test_shot_word_range():
    from paper_2603_14641_b200.dist import shot_word_range
    for shots in [64, 100, 100000]:
        kf = (shots + 63) // 64
        for world in range(1, min(kf, 8) + 1):
            rs = [shot_word_range(shots, world, r) for r in range(world)]
            assert sum(nw for _, nw in rs) == kf
            assert all(rs[i][0] + rs[i][1] == rs[i + 1][0] for i in range(world - 1))


def test_nccl_unique_id_is_128_bytes(q):
    try:
        a = q.nccl_unique_id()
    except q.QuasarError as e:  # NCCL absent: the engine must say so, not fall back
        assert "NCCL" in str(e)
        return
    assert len(a) == 128 and a != q.nccl_unique_id()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2603_14641_b200 import dist as qd
    from paper_2603_14641_b200 import quasar as q
    w, r, _, dist = qd.init_from_env("gloo")
    assert (w, r) == (world, rank)
    try:
        uid = qd.share_nccl_id(dist, rank)
    except q.QuasarError:
        uid = qd.share_bytes(dist, b"x" * 128 if rank == 0 else None)
    # every rank sees rank 0's id
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert all(i == ids[0] for i in ids) and len(uid) == 128
    # max over ranks
    assert qd.max_over_ranks(dist, 1.5 + rank) == 1.5 + world - 1
    # tableau assembly: rank r fills only its generator-word columns of a known tableau
    k = (n + 63) // 64
    rng = np.random.default_rng(7)
    full_x = rng.integers(0, 2**63, size=64 * k * 2 * k, dtype=np.uint64)
    full_s = rng.integers(0, 2**63, size=2 * k, dtype=np.uint64)
    j0, kg = q.shard_range(n, world, rank)
    x = np.zeros_like(full_x)
    s = np.zeros_like(full_s)
    xv, fv = x.reshape(64 * k, 2 * k), full_x.reshape(64 * k, 2 * k)
    xv[:, j0:j0 + kg] = fv[:, j0:j0 + kg]
    xv[:, k + j0:k + j0 + kg] = fv[:, k + j0:k + j0 + kg]
    s[j0:j0 + kg] = full_s[j0:j0 + kg]
    s[k + j0:k + j0 + kg] = full_s[k + j0:k + j0 + kg]
    qd.combine_shard_planes(dist, [x, s])
    np.testing.assert_array_equal(x, full_x)
    np.testing.assert_array_equal(s, full_s)
    dist.barrier()
    dist.destroy_process_group()
    open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")


def test_gloo_two_ranks(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), 1000, str(tmp_path)), nprocs=world, join=True)
    assert sorted(os.listdir(tmp_path)) == ["ok0", "ok1"]
