"""Dataset sharding + per-group loader (paper_2507_13833_b200/loader.py) against the reference's own
shard_dataset / DataLoader (distflow/data_plane.hpp:124-209, compiled into oracle/_ref), and the loader's device
batches against the oracle's generation. Mirrors the reference's loader tests (tests/test_data_plane.cpp)."""
from __future__ import annotations

import os

import numpy as np
import pytest

REF_SO = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libdistflow_ref.so")
need_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")

CASES = [  # dataset size, dp, seed, shuffle, global batch
    (64, 4, 7, False, 16),
    (64, 4, 7, True, 16),
    (96, 2, 11, True, 40),    # per-group 20 over a 48-row shard: wraps inside iteration 2
    (1000, 8, 3, True, 64),
    (30, 3, 5, True, 9),
    (8, 8, 1, True, 8),       # one row per shard
]


def test_shard_dataset_ranges(dfx):
    rs = dfx.shard_dataset(12, 3)
    assert [(r.first, r.last) for r in rs] == [(0, 4), (4, 8), (8, 12)]
    assert all(r.size() == 4 for r in rs)
    with pytest.raises(dfx.errors.IndivisibleError):
        dfx.shard_dataset(10, 3)
    with pytest.raises(dfx.errors.IndivisibleError):
        dfx.shard_dataset(10, 0)


def test_loader_errors(dfx):
    ld = dfx.make_group_loader(16, 4, 1, 9)
    with pytest.raises(dfx.errors.IndivisibleError):
        ld.next_batch_ids(0, 6)
    empty = dfx.DataLoader(dfx.ShardRange(0, 0), 1, 0, 9)
    with pytest.raises(dfx.errors.Error, match="empty"):
        empty.next_batch_ids(0, 4)


def test_loader_is_pure_and_wraps(dfx):
    ld = dfx.make_group_loader(32, 2, 1, 4)  # shard [16, 32), no shuffle
    assert ld.next_batch_ids(0, 8).tolist() == [16, 17, 18, 19]
    assert ld.next_batch_ids(3, 8).tolist() == [28, 29, 30, 31]
    assert ld.next_batch_ids(4, 8).tolist() == [16, 17, 18, 19]  # cursor wraps at the shard end
    assert ld.next_batch_ids(5, 12).tolist() == [30, 31, 16, 17, 18, 19]
    sh = dfx.make_group_loader(32, 2, 1, 4, shuffle=True)
    a = sh.next_batch_ids(0, 32)
    assert sorted(a.tolist()) == list(range(16, 32)) and a.tolist() != list(range(16, 32))  # a permutation
    assert sh.next_batch_ids(0, 32).tolist() == a.tolist()  # pure function of (iteration, batch)


@need_ref
@pytest.mark.parametrize("case", CASES)
def test_loader_ids_match_reference(O, dfx, case):
    n, dp, seed, shuffle, gb = case
    for rank in range(dp):
        ld = dfx.make_group_loader(n, dp, rank, seed, shuffle)
        for it in range(4):
            got = ld.next_batch_ids(it, gb)
            ref = O.ref_loader_ids(n, dp, rank, seed, shuffle, it, gb)
            assert got.dtype == np.uint64 and got.tolist() == ref.tolist(), (case, rank, it)


@need_ref
def test_loader_errors_match_reference(O):
    with pytest.raises(O.OracleError) as e:
        O.ref_loader_ids(10, 3, 0, 1, False, 0, 3)
    assert e.value.kind == O.STATUS_NAMES[3]  # IndivisibleError (dataset size)
    with pytest.raises(O.OracleError) as e:
        O.ref_loader_ids(12, 3, 0, 1, False, 0, 4)
    assert e.value.kind == O.STATUS_NAMES[3]  # IndivisibleError (global batch)


@pytest.mark.gpu
@pytest.mark.parametrize("shuffle", [False, True])
def test_loader_device_batch_bit_exact(O, dfx, shuffle):
    """next_batch -> device PackedBatch: lengths, channels and every token stream equal the oracle's generation
    for the loader's sample ids (duplicates included when the cursor wraps)."""
    import torch
    seed, n_roll = 11, 4
    dist = dfx.TokenDist("uniform", 0, 1, 300)
    ld = dfx.make_group_loader(48, 2, 1, seed, shuffle)
    streams = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward", "token_id")
    for it in (0, 3):
        ids = ld.next_batch_ids(it, 40)  # 20 per group over a 24-row shard: wraps at it = 3
        db = ld.next_batch(it, 40, n_roll, dist, streams=streams)
        torch.cuda.synchronize()
        sb = O.SynthBatch(seed, len(ids), n_roll, O.token_dist("uniform", 1, 1, 300), ids=ids, streams=streams)
        assert db.ids.cpu().numpy().view(np.uint64).tolist() == ids.tolist()
        assert db.host_cu.tolist() == sb.cu_seqlens.tolist()
        T = sb.n_tokens
        for k in streams:
            assert db.streams[k][:T].cpu().numpy().tobytes() == getattr(sb, k)[:T].tobytes(), (it, k)
        assert db.channels["reward"].cpu().numpy().tobytes() == sb.reward.tobytes()


def _loader_worker(rank, world, port, q):
    """One process per DP group (gloo): each rank loads its own shard; the gathered batches must be the ranks'
    reference batches in rank order, and together cover the dataset once per epoch without a shuffle."""
    import torch
    import torch.distributed as dist

    import paper_2507_13833_b200 as d
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        out = []
        for shuffle in (False, True):
            ld = d.make_group_loader(64, world, rank, 13, shuffle)
            for it in range(4):
                mine = torch.from_numpy(ld.next_batch_ids(it, 32).astype("int64"))
                parts = [torch.empty_like(mine) for _ in range(world)]
                dist.all_gather(parts, mine)
                out.append((shuffle, it, [p.tolist() for p in parts]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_loader_gloo_world2(O, dfx):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29300 + (os.getpid() % 400)
    procs = [ctx.Process(target=_loader_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    for e in range(2):  # iterations 2e, 2e+1: 2 groups x 2 x 16 = one pass over the 64 rows (32-row shards)
        epoch = sorted(i for shuffle, it, parts in res[0] if it // 2 == e for part in parts for i in part
                       if not shuffle)
        assert epoch == list(range(64))
    if os.path.exists(REF_SO):
        for shuffle, it, parts in res[0]:
            for r, part in enumerate(parts):
                assert part == O.ref_loader_ids(64, 2, r, 13, shuffle, it, 32).tolist()
