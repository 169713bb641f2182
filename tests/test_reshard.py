"""Reshard (DataBuffer DP m->n) parity.

CPU: the product's native placement (dfx_reshard_placement / segments, csrc/reshard.cu) equals the reference
BufferStore on the 220-config acceptance sweep (golden, from the reference itself); store semantics and errors;
metadata agreement over a world-size-2 gloo group.
GPU: device reshard output serialized with the reference blob format is byte-identical to the reference BufferStore's
get() batches (tests/golden/blobs.npz); the same across 2 GPUs with NCCL P2P (tests/mp/reshard_worker.py).
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_native_placement_matches_reference_sweep(dfx):
    from paper_2507_13833_b200 import reshard as R
    g = np.load(os.path.join(GOLD, "reshard.npz"))
    co = io = 0
    for B, W, dp_p, tp_p, dp_c, tp_c, G in g["cfg"].tolist():
        topo = R.Topology(B, W, tuple([0] * (B * W)))
        dc, idx = R.placement(topo, R.Layout(dp_p, tp_p), R.Layout(dp_c, tp_c), [G // dp_p] * dp_p)
        assert (dc == g["counts"][co:co + dp_c]).all()
        assert (idx == g["ids"][io:io + G]).all()
        # segments reproduce the same index list
        segs = R.segments(topo, R.Layout(dp_p, tp_p), R.Layout(dp_c, tp_c), [G // dp_p] * dp_p)
        rebuilt = np.zeros(G, np.int64)
        dest_base = np.concatenate([[0], np.cumsum(dc.astype(np.int64))]).astype(np.int64)
        for d, p, dr, sr, n in segs:
            rebuilt[dest_base[d] + dr: dest_base[d] + dr + n] = p * (G // dp_p) + sr + np.arange(n)
        assert (rebuilt == idx).all()
        co += dp_c
        io += G


def test_native_placement_errors(dfx):
    from paper_2507_13833_b200 import errors
    from paper_2507_13833_b200 import reshard as R
    t = R.Topology(2, 2, (0, 0, 0, 0))
    with pytest.raises(errors.IndivisibleError):
        R.placement(t, R.Layout(4, 1), R.Layout(2, 2), [1, 2, 1, 2])  # data_plane.hpp:414-416
    with pytest.raises(errors.LayoutError):
        R.placement(R.Topology(2, 3, (0,) * 6), R.Layout(3, 2), R.Layout(6, 1), [2, 2, 2])  # topology.hpp:63-67
    with pytest.raises(errors.LayoutError):
        R.placement(t, R.Layout(3, 1), R.Layout(4, 1), [1, 1, 1])  # dp*tp != world


def test_segments_random_uneven(O, dfx):
    """Uneven producer group sizes: segments == oracle placement (live reference when available)."""
    from paper_2507_13833_b200 import reshard as R
    rng = np.random.default_rng(3)
    for _ in range(50):
        B, W = int(rng.choice([1, 2, 4])), int(rng.choice([2, 4]))
        tp_p, tp_c = int(rng.choice([1, 2])), int(rng.choice([1, 2]))
        dp_p, dp_c = B * W // tp_p, B * W // tp_c
        gc = rng.integers(0, 3, dp_p) * B * W
        try:
            dc, idx = O.reshard_placement(B, W, dp_p, tp_p, dp_c, tp_c, gc)
        except O.OracleError:
            continue
        dc2, idx2 = R.placement(R.Topology(B, W, (0,) * (B * W)), R.Layout(dp_p, tp_p), R.Layout(dp_c, tp_c), gc)
        assert (dc == dc2).all() and (idx == idx2).all()


def test_store_semantics_cpu(dfx):
    """put/ensure_ready bookkeeping and the reference's error types (no device work before exchange)."""
    from paper_2507_13833_b200 import errors
    from paper_2507_13833_b200.reshard import Layout, Topology
    from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan
    topo = Topology(2, 2, (0, 0, 1, 1))
    st = DeviceBufferStore(topo, 0, {"gen": StoreStagePlan(Layout(4, 1), Layout(2, 2))})
    with pytest.raises(errors.UnknownStageError):
        st.put("ghost", 0, 0, 0, None)
    with pytest.raises(errors.Error):  # group 2 lives on rank 1 (data_plane.hpp:249-254)
        st.put("gen", 0, 2, 0, None)
    assert st.put("gen", 0, 0, 0, "b0") is True
    assert st.put("gen", 0, 0, 1, "b0") is False and st.suppressed_count() == 1
    with pytest.raises(errors.Error):  # duplicate (:256-258)
        st.put("gen", 0, 0, 0, "b0")
    with pytest.raises(errors.NotReadyError, match="1 puts outstanding"):
        st.ensure_ready("gen", 0, Layout(2, 2))
    st.worker_done(0)
    st.worker_done(0)  # both local workers done -> low water 1 (:351-367)
    with pytest.raises(errors.StaleIterationError):
        st.put("gen", 0, 1, 0, "b1")
    assert st.put("gen", 1, 1, 0, "b1") is True


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_13833_b200 import reshard as R
        topo = R.Topology.store_per_gpu(world, 2)
        counts = [3 + rank, 3 + rank]  # each rank knows only its own producer groups' sizes
        from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan
        st = DeviceBufferStore(topo, rank, {"s": StoreStagePlan(R.Layout(4, 1), R.Layout(2, 2))},
                               meta_group=torch.distributed.group.WORLD)
        full = [0] * 4
        for j in range(2):
            full[2 * rank + j] = counts[j]
        agreed, sigs = st._agree_counts(full, [2 * rank, 2 * rank + 1], 7 + rank)
        assert sigs == [7, 8]                                 # every rank sees every rank's batch signature
        plan = R.Plan(topo, R.Layout(4, 1), R.Layout(2, 2), [4, 4, 4, 4], rank)
        sends = sorted((i, r) for i, (d, p, *_r) in enumerate(plan.segs) for r in plan.dst_ranks[d]
                       if plan.src_rank[p] == rank and r != rank)
        recvs = sorted((i, plan.src_rank[p]) for i, (d, p, *_r) in enumerate(plan.segs)
                       if rank in plan.dst_ranks[d] and plan.src_rank[p] != rank)
        sizes = np.zeros((len(plan.segs), 2), np.int64)
        for i, (d, p, dr, sr, n) in enumerate(plan.segs):
            if plan.src_rank[p] == rank:
                sizes[i] = (n * 16, n * 1000 + p)
        glob = R.all_reduce_host(sizes, None, torch.distributed.group.WORLD, None)
        q.put((rank, agreed, sends, recvs, glob.tolist(), plan.cross))
    finally:
        torch.distributed.destroy_process_group()


def test_gloo_world2_metadata_agreement(dfx):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == [3, 3, 4, 4]          # every rank sees every producer group's size
    assert res[0][4] == res[1][4]                         # identical global size tables
    assert res[0][5] and res[1][5]                        # dense placement: records cross GPUs
    # what rank 0 sends to rank 1 is exactly what rank 1 expects from rank 0, and vice versa
    assert [i for i, r in res[0][2] if r == 1] == [i for i, s in res[1][3] if s == 0]
    assert [i for i, r in res[1][2] if r == 0] == [i for i, s in res[0][3] if s == 1]


# ---- GPU ----------------------------------------------------------------------------------------
def _blob_of(O, b, d_rec0, d_rec1, streams=("token_id", "lp", "old_lp", "ref_lp")):
    """serialize_records of records [d_rec0, d_rec1) of a device batch (D2H + oracle serializer)."""
    h = b.to_host()
    go = h["group_off"]
    cu = h["cu_seqlens"]
    s0, s1 = int(go[d_rec0]), int(go[d_rec1])
    sub_go = (go[d_rec0:d_rec1 + 1] - s0).astype(np.int32)
    sub_cu = cu[s0:s1 + 1]
    return O.serialize_packed(h["ids"][d_rec0:d_rec1], sub_go, np.diff(sub_cu).astype(np.uint32), sub_cu,
                              [h[k] for k in streams],
                              {"reward": h["reward"][s0:s1], "advantage": h["advantage"][s0:s1]})


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["small", "cross", "dense"])
def test_device_reshard_blobs_bit_exact_single_gpu(O, dfx, name):
    from paper_2507_13833_b200 import reshard as R
    g = np.load(os.path.join(GOLD, "blobs.npz"))
    B, W, dp_p, tp_p, dp_c, tp_c = (int(x) for x in g[f"{name}_cfg"])
    sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48),
                      streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
    T = sb.n_tokens
    b = dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward},
                                  {k: getattr(sb, k)[:T] for k in ("token_id", "lp", "old_lp", "ref_lp", "mask")})
    dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, dfx.StageContext())
    topo = R.Topology(B, W, tuple([0] * (B * W)))  # every logical worker on this GPU
    per = 16 // dp_p
    plan = R.Plan(topo, R.Layout(dp_p, tp_p), R.Layout(dp_c, tp_c), [per] * dp_p, 0)
    sources = {p: (b.view_records(p * per, (p + 1) * per), 0) for p in range(dp_p)}
    cb = R.exchange(plan, sources)
    torch.cuda.synchronize()
    assert cb.groups == list(range(dp_c))
    ids = cb.batch.ids.cpu().numpy().view(np.uint64)
    assert (ids == g[f"{name}_ids"]).all()
    for i, d in enumerate(cb.groups):
        blob = _blob_of(O, cb.batch, cb.rec_off[i], cb.rec_off[i + 1])
        assert blob.tobytes() == g[f"{name}_blob_{d}"].tobytes(), f"dest {d}"


@pytest.mark.gpu
def test_device_reshard_materialized_copy(O, dfx):
    """Non-contiguous placement on one GPU forces the copy path (device copies + unpack kernel)."""
    from paper_2507_13833_b200 import reshard as R
    sb = O.SynthBatch(3, 32, 4, O.token_dist("uniform", 0, 1, 300), streams=("lp", "old_lp", "ref_lp", "mask"))
    T = sb.n_tokens
    b = dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward},
                                  {k: getattr(sb, k)[:T] for k in ("lp", "old_lp", "ref_lp", "mask")})
    topo = R.Topology(2, 2, (0, 0, 0, 0))
    plan = R.Plan(topo, R.Layout(4, 1), R.Layout(2, 2), [8] * 4, 0)
    cb = R.exchange(plan, {p: (b.view_records(8 * p, 8 * p + 8), 0) for p in range(4)})
    assert not cb.zero_copy
    _, idx = O.reshard_placement(2, 2, 4, 1, 2, 2, [8] * 4)
    assert (cb.batch.ids.cpu().numpy().view(np.uint64) == sb.ids[idx]).all()
    # token streams of each destination record equal the source record's
    cb.batch.ensure_host_meta()
    go, cu = cb.batch.host_group_off, cb.batch.host_cu
    lp = cb.batch.streams["lp"].cpu().numpy()
    for k, r in enumerate(idx.tolist()):
        for j in range(4):
            s_src, s_dst = 4 * r + j, go[k] + j
            a = sb.lp[sb.cu_seqlens[s_src]:sb.cu_seqlens[s_src + 1]]
            assert lp[cu[s_dst]:cu[s_dst + 1]].tobytes() == a.tobytes()
    # the loss on the resharded batch equals the loss on the original (same records, new order)
    ctx = dfx.StageContext()
    a = dfx.loss_dict(dfx.ppo_loss(b, ctx, adv_source="group")["out"][0])
    c = dfx.loss_dict(dfx.ppo_loss(cb.batch, ctx, adv_source="group")["out"][0])
    assert a["n_tokens"] == c["n_tokens"] and abs(a["loss"] - c["loss"]) < 1e-9


@pytest.mark.gpu
def test_two_gpu_nccl_reshard():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = 29600 + (os.getpid() % 500)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp", "reshard_worker.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("RESHARD_OK") == 2, r.stdout[-2000:]


@pytest.mark.gpu
def test_two_gpu_lazy_reshard_fused_loss():
    """TP partners on different GPUs: the loss kernel reading the partner's records over NVLink in place equals
    the loss over the materialized consumer batch (tests/mp/lazy_loss_worker.py)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = 29100 + (os.getpid() % 500)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp", "lazy_loss_worker.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("LAZY_OK") == 2, r.stdout[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [1, 2, 4])
def test_native_dstore_blobs(n_gpus):
    """The native distributed DataBuffer (libdfx dfx_dstore_*: one process per GPU, NCCL) reproduces the reference
    BufferStore's destination blobs byte for byte, and the round trip gives back the producers' records
    (tests/mp/dstore_worker.py)."""
    if torch.cuda.device_count() < n_gpus:
        pytest.skip(f"needs {n_gpus} GPUs")
    port = 27600 + n_gpus * 50 + (os.getpid() % 40)
    r = subprocess.run(["timeout", "300", sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n_gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp", "dstore_worker.py")],
                       capture_output=True, text=True, timeout=360, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("DSTORE_OK") == n_gpus, r.stdout[-2000:]
    print(r.stdout[-1500:])


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [2, 4])
def test_mixed_zero_copy_lazy_reshard(n_gpus):
    """Zero-copy and peer-reading GPUs in one lazy reshard, several iterations over the same producer batches and a
    collective in between: no deadlock, every group's loss equals the oracle, peer mappings do not accumulate
    (tests/mp/mixed_lazy_worker.py)."""
    if torch.cuda.device_count() < n_gpus:
        pytest.skip(f"needs {n_gpus} GPUs")
    port = 28600 + n_gpus * 50 + (os.getpid() % 40)
    r = subprocess.run(["timeout", "300", sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n_gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp", "mixed_lazy_worker.py")],
                       capture_output=True, text=True, timeout=360, cwd=ROOT)
    errs = "\n".join(l for l in r.stderr.splitlines() if "Error" in l or "assert" in l)[-4000:]
    assert r.returncode == 0, r.stdout[-2000:] + errs
    assert r.stdout.count("MIXED_OK") == n_gpus, r.stdout[-2000:]
    print(r.stdout[-1500:])


def _metrics_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2507_13833_b200 as dfx
        stats = torch.tensor([3.0 + rank, 1.5 * (rank + 1), 2.0 + rank], dtype=torch.float64)
        q.put((rank, dfx.aggregate_metrics(stats, tokens=100 * (rank + 1), suppressed=rank)))
    finally:
        dist.destroy_process_group()


def test_aggregate_metrics_gloo_world2(dfx):
    """aggregate_metrics (worker.hpp:275-325) as one all-reduce: totals and reward mean/variance like rank 0 of
    the reference computes them from the gathered per-rank sums."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 500)
    procs = [ctx.Process(target=_metrics_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, s, sq = 3.0 + 4.0, 1.5 + 3.0, 2.0 + 3.0
    want = {"reward_count": 7, "reward_mean": s / n, "reward_variance": sq / n - (s / n) ** 2, "global_tokens": 300,
            "suppressed_total": 1}
    assert res[0] == res[1] == want
