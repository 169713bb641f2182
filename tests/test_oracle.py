"""CPU tests: pin the oracle (oracle/dfx_oracle.c) to the reference's own known answers and golden fixtures.

- known-answer tests re-hosted from the reference's GoogleTest suites (file:line cited per test)
- golden fixtures in tests/golden/*.npz, produced by running the reference itself (tests/golden/make_golden.py)
- where the compiled reference (oracle/_ref) is present, live randomized comparisons
"""
from __future__ import annotations

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


# ---- hash (tests/test_hash.cpp) ------------------------------------------------------------
def test_splitmix_known_values(O):
    gamma = 0x9E3779B97F4A7C15  # tests/test_hash.cpp:10-17
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.splitmix64(gamma) == 0x6E789E6AA1B965F4
    assert O.splitmix64((gamma * 2) % 2**64) == 0x06C45D188009454F


def test_keyed_hash_key_sensitivity(O):
    a = O.keyed_hash(1, "reward", 7, 3)  # tests/test_hash.cpp:19-26
    assert a == O.keyed_hash(1, "reward", 7, 3)
    assert a != O.keyed_hash(2, "reward", 7, 3)
    assert a != O.keyed_hash(1, "value", 7, 3)
    assert a != O.keyed_hash(1, "reward", 8, 3)
    assert a != O.keyed_hash(1, "reward", 7, 4)


def test_unit_and_symmetric_ranges(O):
    u = [O.unit_from_hash(O.keyed_hash(42, "reward", i)) for i in range(10000)]  # test_hash.cpp:28-47
    assert min(u) >= 0.0 and max(u) < 1.0
    v = [O.symmetric_from_hash(O.keyed_hash(42, "value", i)) for i in range(10000)]
    assert min(v) >= -1.0 and max(v) <= 1.0 and min(v) < -0.5 and max(v) > 0.5


def test_hash_bytes(O):
    b1 = O.hash_bytes(123, 1024)  # test_hash.cpp:49-57
    assert (b1 == O.hash_bytes(123, 1024)).all() and len(set(b1.tolist())) > 64
    assert not (b1 == O.hash_bytes(124, 1024)).all()


def test_hash_golden(O):
    g = gold("hash.npz")
    assert [O.splitmix64(int(z)) for z in g["z"]] == g["splitmix"].tolist()
    for i in range(len(g["keyed"])):
        h = O.keyed_hash(int(g["kh_seed"][i]), str(g["kh_dom"][i]), int(g["kh_a"][i]), int(g["kh_b"][i]))
        assert h == int(g["keyed"][i])
        assert O.unit_from_hash(h) == g["unit"][i] and O.symmetric_from_hash(h) == g["sym"][i]
    assert [O.keyed_hash(1, "tok_lp", 5, 2, t) for t in range(16)] == g["keyed3"].tolist()
    assert (O.hash_bytes(123, 1027) == g["hash_bytes_123"]).all()


# ---- generation (tests/test_functions.cpp:45-132) -------------------------------------------
def test_generation_golden(O):
    g = gold("generation.npz")
    ids = g["ids"]
    for name in ("const", "uniform", "c2", "small"):
        seed, kind, val, lo, hi, n_roll, bpt = (int(x) for x in g[f"{name}_params"])
        sb = O.SynthBatch(seed, len(ids), n_roll, O.TokenDist(kind, val, lo, hi), ids=ids, streams=())
        assert (np.diff(sb.cu_seqlens) == g[f"{name}_tokens"]).all(), name
        if bpt:  # fn_generate payload = hash_bytes(keyed_hash(seed, "payload", id, r), tokens * bpt)
            pay = []
            for r, sid in enumerate(ids):
                for j in range(n_roll):
                    L = int(g[f"{name}_tokens"][r * n_roll + j])
                    pay.append(O.hash_bytes(O.keyed_hash(seed, "payload", int(sid), j), L * bpt))
            assert (np.concatenate(pay) == g[f"{name}_payload"]).all(), name
    sb = O.SynthBatch(11, len(ids), 4, O.token_dist("constant", 1), ids=ids, streams=())
    assert sb.reward.tobytes() == g["reward"].tobytes()  # fill_channel, unit range
    assert sb.value.tobytes() == g["value"].tobytes()    # fill_channel, symmetric


def test_generation_properties(O):
    sb = O.SynthBatch(5, 16, 4, O.token_dist("uniform", 0, 16, 48), streams=())  # test_functions.cpp:57-80
    L = np.diff(sb.cu_seqlens)
    assert len(L) == 64 and L.min() >= 16 and L.max() <= 48 and len(set(L.tolist())) > 1
    sk = O.SynthBatch(11, 4096, 16, O.token_dist("skewed", 0, 1, 16384), streams=())
    L = np.diff(sk.cu_seqlens)
    assert L.min() >= 1 and L.max() <= 16384 and np.median(L) < L.mean()  # skewed toward short, long tail
    r = O.SynthBatch(11, 5000, 2, O.token_dist("constant", 1), streams=()).reward  # test_functions.cpp:101-132
    assert abs(r.mean() - 0.5) < 0.02 and abs(r.var() - 1 / 12) < 0.01


def test_token_streams_properties(O):
    sb = O.SynthBatch(1, 64, 8, O.token_dist("constant", 1024))
    T = sb.n_tokens
    assert T == 64 * 8 * 1024
    assert (sb.lp[:T] <= 0).all() and (sb.lp[:T] >= -4).all()
    assert np.abs(sb.old_lp[:T] - sb.lp[:T]).max() <= 0.25 + 1e-6
    assert np.abs(sb.ref_lp[:T] - sb.lp[:T]).max() <= 0.1 + 1e-6
    assert 0.85 < sb.mask[:T].mean() < 0.95  # ~10% masked prompt prefix
    # deterministic and thread-count independent
    sb1 = O.SynthBatch(1, 64, 8, O.token_dist("constant", 1024), nthreads=1)
    assert sb1.lp.tobytes() == sb.lp.tobytes() and sb1.mask.tobytes() == sb.mask.tobytes()


# ---- advantages (tests/test_functions.cpp:134-192) -----------------------------------------------
def test_group_advantage_kats(O):
    assert O.grpo_advantage([0, 4], [1.0, 0.0, 1.0, 0.0], 0.0).tolist() == [1.0, -1.0, 1.0, -1.0]
    z = O.grpo_advantage([0, 3], [0.75, 0.75, 0.75], 0.0)
    assert z.tolist() == [0.0, 0.0, 0.0]
    assert O.grpo_advantage([0, 2], [1.0, 0.0], 0.0)[0] > O.grpo_advantage([0, 2], [1.0, 0.0], 0.5)[0]
    with pytest.raises(O.OracleError) as e:
        O.grpo_advantage([0, 0], [], 0.0)
    assert e.value.kind == "MissingRolloutsError"


def test_ppo_advantage_kat(O):
    assert O.ppo_advantage([0.9, 0.2], [0.4, -0.1]).tolist() == [0.9 - 0.4, 0.2 - (-0.1)]


def test_advantage_golden_bit_exact(O):
    g = gold("advantage.npz")
    for eps in (0.0, 1e-6, 0.5):
        assert O.grpo_advantage(g["group_off"], g["reward"], eps).tobytes() == g[f"grpo_eps_{eps}"].tobytes()
    assert O.ppo_advantage(g["reward"], g["value"]).tobytes() == g["ppo"].tobytes()


# ---- GAE / loss known answers (our convention; parity unpinned upstream) ------------------------------
def test_gae_kat(O):
    cu = np.array([0, 3, 5], np.int64)
    r = np.array([0, 0, 1, 0, 2], np.float32)
    v = np.array([0.5, 0.5, 0.5, 1.0, -1.0], np.float32)
    m = np.array([1, 1, 1, 0, 1], np.uint8)
    A, R, ws = O.gae(cu, r, v, m, gamma=1.0, lam=0.5)
    # seq 0: delta = [0, 0, .5] -> A = [.125, .25, .5]
    assert A[:3].tolist() == [0.125, 0.25, 0.5] and R[:3].tolist() == [0.625, 0.75, 1.0]
    # seq 1: t=4 last: delta = 2 - (-1) = 3, A4 = 3; t=3: m1 = 1, v1 = -1: delta = 0 + (-1) - 1 = -2, A3 = -2 + .5*3
    assert A[3:].tolist() == [-0.5, 3.0]
    assert ws.tolist() == [0.125 + 0.25 + 0.5 + 3.0, 0.125**2 + 0.25**2 + 0.25 + 9.0, 4.0]


def test_loss_kat(O):
    cu = np.array([0, 2], np.int64)
    lp = np.array([-1.0, -2.0], np.float32)
    old = np.array([-1.0, -2.5], np.float32)   # ratios 1 and e^0.5 = 1.6487 (> 1.2: clipped for A > 0)
    ref = np.array([-1.0, -2.0], np.float32)   # KL 0
    adv = np.array([1.0, 1.0], np.float32)
    m = np.array([1, 1], np.uint8)
    out, g = O.ppo_loss(cu, lp, old, ref, adv, m, O.loss_cfg(beta=0.0), want_grad=True)
    # pg = max(-A rho, -A clip) : token0 = -1, token1 = max(-1.6487, -1.2) = -1.2 (clipped)
    assert abs(out["pg_loss"] - (-1.0 - 1.2) / 2) < 1e-15
    assert out["clipfrac"] == 0.5 and out["n_tokens"] == 2 and out["kl"] == 0.0
    assert abs(g[0] - (-1.0 / 2)) < 1e-15 and g[1] == 0.0  # clipped token carries no gradient
    out2, _ = O.ppo_loss(cu, lp, old, ref, -adv, m, O.loss_cfg(beta=0.0))
    # A < 0: pg = max(rho, min-clip ...) -> token0 = 1, token1 = max(1.6487, 1.2) = 1.6487 (unclipped)
    assert abs(out2["pg_loss"] - (1.0 + np.exp(0.5)) / 2) < 1e-7 and out2["clipfrac"] == 0.0
    # k3 KL with ref = lp + 0.1: e^0.1 - 0.1 - 1
    out3, _ = O.ppo_loss(cu, lp, lp, lp + np.float32(0.1), adv * 0, m, O.loss_cfg(beta=1.0, kl="k3"))
    x = np.float64(np.float32(lp[0] + np.float32(0.1))) - np.float64(lp[0])
    assert abs(out3["kl"] - (np.exp(x) - x - 1)) < 1e-9


def test_loss_aggregations(O):
    cu = np.array([0, 1, 4], np.int64)
    lp = np.zeros(4, np.float32)
    adv = np.array([1.0, 2.0, 2.0, 2.0], np.float32)
    m = np.ones(4, np.uint8)
    tm, _ = O.ppo_loss(cu, lp, lp, lp, adv, m, O.loss_cfg(beta=0.0, agg="token-mean"))
    sm, _ = O.ppo_loss(cu, lp, lp, lp, adv, m, O.loss_cfg(beta=0.0, agg="seq-mean-token-mean"))
    ss, _ = O.ppo_loss(cu, lp, lp, lp, adv, m, O.loss_cfg(beta=0.0, agg="seq-mean-token-sum"))
    assert tm["pg_loss"] == -7 / 4 and sm["pg_loss"] == (-1 - 2) / 2 and ss["pg_loss"] == (-1 - 6) / 2


# ---- record blob (tests/test_record.cpp) ------------------------------------------------------------
def test_blob_size_arithmetic_and_layout(O):
    # one record, one rollout, 8-byte payload, channel "reward": 4 + 16 + 42 (test_record.cpp:108-121)
    payload = np.full(8, 0x55, np.uint8)
    b = O.serialize_packed([1], [0, 1], [2], [0, 8], [payload], {"reward": np.array([1.0])})
    assert len(b) == 4 + 16 + 42
    assert b[:4].tolist() == [1, 0, 0, 0]            # LE u32 record count (test_record.cpp:155-166)
    assert b[4:12].tolist() == [1, 0, 0, 0, 0, 0, 0, 0]


def test_blob_golden_and_channel_order(O):
    g = gold("blobs.npz")
    sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48), streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
    T = sb.n_tokens
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    assert adv.tobytes() == g["adv"].tobytes()
    streams = [sb.token_id[:T], sb.lp[:T], sb.old_lp[:T], sb.ref_lp[:T]]
    # channel dict order must not matter: std::map order (test_record.cpp:138-153)
    b1 = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, streams,
                            {"reward": sb.reward, "advantage": adv})
    b2 = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, streams,
                            {"advantage": adv, "reward": sb.reward})
    assert b1.tobytes() == b2.tobytes() == g["blob"].tobytes()


# ---- reshard placement (tests/test_data_plane.cpp, tests/acceptance_test.cpp) ---------------------------
def test_reshard_fig8_walkthrough(O):
    # 1 node x 4 workers, dp2 tp2 -> dp4: group g gets ids g*16.. (test_data_plane.cpp:175-204)
    dc, idx = O.reshard_placement(1, 4, 2, 2, 4, 1, [32, 32])
    assert dc.tolist() == [16] * 4 and idx.tolist() == list(range(64))


def test_reshard_cross_node_swap(O):
    # 2 x 4, dp2 tp4 -> dp8: store0 = a0..a15, b0..b15 ; store1 = a16..a31, b16..b31 (test_data_plane.cpp:219-263)
    dc, idx = O.reshard_placement(2, 4, 2, 4, 8, 1, [32, 32])
    assert dc.tolist() == [8] * 8
    store0 = idx[:32].tolist()
    store1 = idx[32:].tolist()
    assert store0 == list(range(16)) + list(range(32, 48))
    assert store1 == list(range(16, 32)) + list(range(48, 64))


def test_reshard_fast_path_and_errors(O):
    dc, idx = O.reshard_placement(2, 2, 4, 1, 4, 1, [8, 8, 8, 8])  # unchanged dp: identity (:265-288)
    assert idx.tolist() == list(range(32))
    with pytest.raises(O.OracleError) as e:
        O.reshard_placement(2, 2, 4, 1, 2, 2, [1, 2, 1, 2])  # store holds 3 records, B = 2 (data_plane.hpp:414-416)
    assert e.value.kind == "IndivisibleError"
    with pytest.raises(O.OracleError) as e:
        O.reshard_placement(2, 3, 3, 2, 6, 1, [2, 2, 2])  # tp 2 does not divide W 3 (topology.hpp:63-67)
    assert e.value.kind == "LayoutError"


def test_reshard_220_configs_golden(O):
    """Oracle placement == the reference BufferStore on the acceptance sweep (acceptance_test.cpp:183-254)."""
    g = gold("reshard.npz")
    co = io = 0
    for B, W, dp_p, tp_p, dp_c, tp_c, G in g["cfg"].tolist():
        dc, idx = O.reshard_placement(B, W, dp_p, tp_p, dp_c, tp_c, np.full(dp_p, G // dp_p, np.uint64))
        assert (dc == g["counts"][co:co + dp_c]).all()
        assert (idx == g["ids"][io:io + G]).all()
        assert sorted(idx.tolist()) == list(range(G))  # multiset preserved, counts G/dp_c
        assert (dc == G // dp_c).all()
        co += dp_c
        io += G


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                    "libdistflow_ref.so")), reason="compiled reference absent")
def test_live_reference_random(O):
    rng = np.random.default_rng(7)
    for _ in range(30):
        n = int(rng.integers(1, 40))
        sizes = rng.integers(1, 9, n).astype(np.int32)
        go = np.zeros(n + 1, np.int32)
        np.cumsum(sizes, out=go[1:])
        reward = rng.integers(0, 3, int(go[-1])).astype(np.float64) / 2
        out = np.zeros(int(go[-1]))
        assert O.ref().ref_advantage(0, n, O.ptr(go), O.ptr(reward), None, 1e-6, O.ptr(out)) == 0
        assert O.grpo_advantage(go, reward, 1e-6).tobytes() == out.tobytes()
    for _ in range(30):  # random uneven group counts through the reference store
        B = int(rng.choice([1, 2, 4]))
        W = int(rng.choice([2, 4]))
        tp_p, tp_c = int(rng.choice([1, 2])), int(rng.choice([1, 2]))
        dp_p, dp_c = B * W // tp_p, B * W // tp_c
        per = int(rng.integers(1, 4)) * B * (W // tp_c)
        gc = np.full(dp_p, per, np.uint64)
        G = int(gc.sum())
        try:
            dc, idx = O.reshard_placement(B, W, dp_p, tp_p, dp_c, tp_c, gc)
        except O.OracleError as e:
            with pytest.raises(O.OracleError) as e2:
                O.ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, gc, np.arange(G, dtype=np.uint64))
            assert e2.value.kind == e.kind
            continue
        dc2, did, _, _ = O.ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, gc, np.arange(G, dtype=np.uint64))
        assert (dc == dc2).all() and (idx == did).all()


@pytest.mark.parametrize("agg", [0, 1, 2])
def test_loss_port_threads_match_single_thread(O, agg):
    """bench.py's CPU baseline times dfo_ppo_loss_mt; it must compute what the single-thread checker computes."""
    sb = O.SynthBatch(5, 24, 4, O.token_dist("uniform", 0, 1, 700), streams=("lp", "old_lp", "ref_lp", "mask"))
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    at = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    cfg = O.loss_cfg()
    cfg.agg = agg
    a, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, at, sb.mask, cfg)
    for nt in (2, 7, 200):
        b = O.ppo_loss_mt(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, at, sb.mask, cfg, nt)
        for k in a:
            assert abs(a[k] - b[k]) <= 1e-12 * max(1.0, abs(a[k])), (nt, k, a[k], b[k])
