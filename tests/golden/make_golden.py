"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

The reference is compiled from /root/reference/proj/include (unmodified headers) into oracle/_ref by
oracle/Makefile; this script calls its entry points (oracle/ref_shim.cpp) and stores inputs + outputs as .npz so the
oracle and the CUDA path can be checked where /root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py     # needs oracle/_ref/libdistflow_ref.so
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def hashes():
    R = O.ref()
    gamma = 0x9E3779B97F4A7C15
    z = np.array([0, gamma, (gamma * 2) % 2**64, 1, 12345, 2**64 - 1], np.uint64)
    sm = np.array([R.ref_splitmix64(int(v)) for v in z], np.uint64)
    tuples = [(1, "reward", 7, 3), (2, "reward", 7, 3), (1, "value", 7, 3), (1, "reward", 8, 3), (1, "reward", 7, 4),
              (42, "gen_tokens", 100, 15), (11, "tok_lp", 5, 2)]
    kh = np.array([R.ref_keyed_hash2(s, d.encode(), a, b) for s, d, a, b in tuples], np.uint64)
    kh3 = np.array([R.ref_keyed_hash3(1, b"tok_lp", 5, 2, t) for t in range(16)], np.uint64)
    unit = np.array([R.ref_unit_from_hash(int(h)) for h in kh], np.float64)
    sym = np.array([R.ref_symmetric_from_hash(int(h)) for h in kh], np.float64)
    hb = np.zeros(1027, np.uint8)
    R.ref_hash_bytes(123, O.ptr(hb), hb.size)
    np.savez(os.path.join(HERE, "hash.npz"), z=z, splitmix=sm, kh_seed=np.array([t[0] for t in tuples], np.uint64),
             kh_dom=np.array([t[1] for t in tuples]), kh_a=np.array([t[2] for t in tuples], np.uint64),
             kh_b=np.array([t[3] for t in tuples], np.uint64), keyed=kh, keyed3=kh3, unit=unit, sym=sym,
             hash_bytes_123=hb)


def generation():
    R = O.ref()
    out = {}
    ids = np.arange(0, 96, dtype=np.uint64) * 7 + 3
    for name, kind, val, lo, hi, n_roll, bpt, seed in [("const", 0, 128, 0, 0, 1, 2, 5), ("uniform", 1, 0, 16, 48, 4, 3, 5),
                                                       ("c2", 1, 0, 1, 4096, 16, 0, 1), ("small", 1, 0, 16, 48, 2, 2, 7)]:
        tc = np.zeros(len(ids) * n_roll, np.uint32)
        pl = np.zeros(int(tc.size) * 4096 * 3 if bpt else 1, np.uint8)
        assert R.ref_generate(seed, kind, val, lo, hi, n_roll, bpt, O.ptr(ids), len(ids), O.ptr(tc),
                              O.ptr(pl) if bpt else None) == 0
        out[f"{name}_tokens"] = tc
        out[f"{name}_params"] = np.array([seed, kind, val, lo, hi, n_roll, bpt], np.int64)
        if bpt:
            out[f"{name}_payload"] = pl[: int(tc.astype(np.int64).sum()) * bpt]
    rw, vl, rl = (np.zeros(len(ids) * 4) for _ in range(3))
    assert R.ref_fill_channels(11, O.ptr(ids), len(ids), 4, O.ptr(rw), O.ptr(vl), O.ptr(rl)) == 0
    np.savez(os.path.join(HERE, "generation.npz"), ids=ids, reward=rw, value=vl, ref_logprob=rl, **out)


def advantages():
    R = O.ref()
    rng = np.random.default_rng(2024)
    sizes = rng.integers(1, 20, 300).astype(np.int32)
    go = np.zeros(len(sizes) + 1, np.int32)
    np.cumsum(sizes, out=go[1:])
    S = int(go[-1])
    reward = rng.random(S)
    # ties, equal groups and binary rewards (the KAT shapes of tests/test_functions.cpp:134-168)
    for g in range(0, 300, 7):
        reward[go[g]:go[g + 1]] = 0.75
    for g in range(3, 300, 11):
        reward[go[g]:go[g + 1]] = rng.integers(0, 2, go[g + 1] - go[g]).astype(np.float64)
    value = rng.random(S) * 2 - 1
    res = {}
    for eps in (0.0, 1e-6, 0.5):
        adv = np.zeros(S)
        assert R.ref_advantage(0, len(sizes), O.ptr(go), O.ptr(reward), None, eps, O.ptr(adv)) == 0
        res[f"grpo_eps_{eps}"] = adv
    ppo = np.zeros(S)
    assert R.ref_advantage(1, len(sizes), O.ptr(go), O.ptr(reward), O.ptr(value), 0.0, O.ptr(ppo)) == 0
    np.savez(os.path.join(HERE, "advantage.npz"), group_off=go, reward=reward, value=value, ppo=ppo, **res)


def reshard_configs():
    """The acceptance property sweep's shape (tests/acceptance_test.cpp:183-254): random (B, W, tp_p, tp_c, G)."""
    rng = np.random.default_rng(912662)
    rows, counts, ids, stats = [], [], [], []
    for trial in range(220):
        B = [1, 2, 4][rng.integers(3)]
        W = [2, 4][rng.integers(2)]
        tp_p = [1, 2][rng.integers(2)]
        tp_c = [1, 2][rng.integers(2)]
        world = B * W
        step = np.lcm(world, B * B)
        kmin, kmax = (8 + step - 1) // step, 256 // step
        G = int(step * (kmin + rng.integers(kmax - kmin + 1)))
        dp_p, dp_c = world // tp_p, world // tp_c
        gc = np.full(dp_p, G // dp_p, np.uint64)
        dc, did, _, st = O.ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, gc, np.arange(G, dtype=np.uint64))
        rows.append([B, W, dp_p, tp_p, dp_c, tp_c, G])
        counts.append(dc)
        ids.append(did)
        stats.append(st)
    np.savez(os.path.join(HERE, "reshard.npz"), cfg=np.array(rows, np.int64),
             counts=np.concatenate(counts), ids=np.concatenate(ids), stats=np.concatenate(stats))


def blobs():
    """serialize_records of a packed batch, and the per-destination blobs of a full reference reshard."""
    sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48), streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
    T = sb.n_tokens
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    streams = [sb.token_id[:T], sb.lp[:T], sb.old_lp[:T], sb.ref_lp[:T]]
    ch = {"reward": sb.reward, "advantage": adv}
    blob = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, streams, ch, use_reference=True)
    out = {"blob": blob, "adv": adv}
    # reshard dp 4 (tp 1) -> dp 2 (tp 2) on 1 node x 4 workers (configs/grpo_small.json layouts), and
    # dp 4 -> dp 8 on 2 nodes x 4 workers (tp 2 -> tp 1)
    for name, (B, W, dp_p, tp_p, dp_c, tp_c) in {"small": (1, 4, 4, 1, 2, 2), "cross": (2, 4, 4, 2, 8, 1),
                                                  "dense": (2, 2, 4, 1, 2, 2)}.items():
        gc = np.full(dp_p, 16 // dp_p, np.uint64)
        dc, did, bl, st = O.ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, gc, sb.ids, sb.group_off, sb.tok_count,
                                        sb.cu_seqlens, streams, ch, want_blobs=True, blob_cap=1 << 22)
        out[f"{name}_cfg"] = np.array([B, W, dp_p, tp_p, dp_c, tp_c], np.int64)
        out[f"{name}_counts"] = dc
        out[f"{name}_ids"] = did
        out[f"{name}_stats"] = st
        for d, b in enumerate(bl):
            out[f"{name}_blob_{d}"] = b
    np.savez(os.path.join(HERE, "blobs.npz"), **out)


if __name__ == "__main__":
    O.lib()
    O.ref()
    hashes()
    generation()
    advantages()
    reshard_configs()
    blobs()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
