"""Synthetic rollout metadata on the host (lengths, rollout channels), vectorised over rollouts.

Restates the reference's generation path so the product can build batches without the oracle:
keyed SplitMix64 (distflow/hash.hpp:14-45), draw_tokens (distflow/functions.hpp:67-80) plus the SKEWED
kind, and fill_channel for reward/value (distflow/functions.hpp:95-104, 130-138).
Per-token streams are generated on the device by dfx_synth_tokens (csrc/synth.cu).
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def hash_combine(seed, v):
    seed = np.asarray(seed, dtype=np.uint64)
    v = np.asarray(v, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(seed ^ (v + GAMMA + (seed << np.uint64(6)) + (seed >> np.uint64(2))))


def hash_str(seed: int, s: str):
    h = np.uint64(seed)
    for ch in s.encode():
        h = hash_combine(h, ch)
    return np.uint64(h)


def keyed_hash(seed: int, domain: str, *counters):
    h = hash_str(seed, domain)
    for c in counters:
        h = hash_combine(h, c)
    return h


def unit_from_hash(h):
    return (np.asarray(h, np.uint64) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def symmetric_from_hash(h):
    return 2.0 * unit_from_hash(h) - 1.0


class TokenDist:
    """distflow::TokenDist (functions.hpp:19-24) + SKEWED (product of three 21-bit uniforms)."""

    KINDS = ("constant", "uniform", "skewed")

    def __init__(self, kind: str = "constant", value: int = 128, min: int = 64, max: int = 192):  # noqa: A002
        if kind not in self.KINDS:
            raise ValueError(f"unknown token distribution '{kind}'")
        self.kind, self.value, self.min, self.max = kind, int(value), int(min), int(max)

    def draw(self, seed: int, sample_ids, rollouts) -> np.ndarray:
        """draw_tokens for arrays of (sample_id, rollout)."""
        ids = np.asarray(sample_ids, np.uint64)
        rs = np.asarray(rollouts, np.uint64)
        if self.kind == "constant":
            return np.full(np.broadcast(ids, rs).shape, self.value, np.int64)
        if self.max < self.min:
            raise ValueError("token distribution max < min")  # functions.hpp:73
        span = self.max - self.min + 1
        h = hash_combine(hash_combine(hash_str(seed, "gen_tokens"), ids), rs)
        if self.kind == "uniform":
            return self.min + (h % np.uint64(span)).astype(np.int64)
        mask21 = np.uint64(0x1FFFFF)
        with np.errstate(over="ignore"):
            prod = (h & mask21) * ((h >> np.uint64(21)) & mask21) * ((h >> np.uint64(42)) & mask21)
        # floor(span * prod / 2^63) with 128-bit intermediate: split prod into 32-bit halves
        hi = prod >> np.uint64(32)
        lo = prod & np.uint64(0xFFFFFFFF)
        sp = np.uint64(span)
        with np.errstate(over="ignore"):
            a = hi * sp                       # < 2^31 * 2^32
            b = lo * sp                       # < 2^32 * 2^32 (may wrap: keep carry separately)
        # span*prod = a*2^32 + b ; (>>63) = (a*2^32 + b) >> 63 = (a + (b >> 32)) >> 31 exactly
        q = (a + (b >> np.uint64(32))) >> np.uint64(31)
        return self.min + q.astype(np.int64)


def rollout_lengths(seed: int, ids, n_roll: int, dist: TokenDist) -> np.ndarray:
    ids = np.asarray(ids, np.uint64)
    rid = np.repeat(ids, n_roll)
    rr = np.tile(np.arange(n_roll, dtype=np.uint64), len(ids))
    return dist.draw(seed, rid, rr)


def rollout_channels(seed: int, ids, n_roll: int):
    """fn_reward (unit range) and fn_value (symmetric) per rollout, as fill_channel computes them."""
    ids = np.asarray(ids, np.uint64)
    rid = np.repeat(ids, n_roll)
    rr = np.tile(np.arange(n_roll, dtype=np.uint64), len(ids))
    reward = unit_from_hash(hash_combine(hash_combine(hash_str(seed, "reward"), rid), rr))
    value = symmetric_from_hash(hash_combine(hash_combine(hash_str(seed, "value"), rid), rr))
    return reward, value


def generate_rollouts(seed: int, ids, n_roll: int, dist: TokenDist, bytes_per_token: int, stream=None):
    """fn_generate (functions.hpp:108-123) on the device: per-rollout token counts (draw_tokens) and the
    concatenated hash_bytes payloads (hash.hpp:48-59), bit-identical to the reference.
    ids: device uint64/int64 tensor [R]. Returns (tok_count u32 [R*n_roll], payload_off i64 [R*n_roll+1],
    payload u8 [total]) on the device. One host synchronisation (the payload size)."""
    import ctypes as C

    import torch

    from . import _abi

    if n_roll < 1:
        raise ValueError("rollouts_per_prompt must be >= 1")  # functions.hpp:111
    L = _abi.lib()
    R = int(ids.numel())
    S = R * n_roll
    dev = ids.device
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    kind = TokenDist.KINDS.index(dist.kind)
    counts = torch.empty(max(S, 1), dtype=torch.int32, device=dev)
    _abi.check(L.dfx_generate_counts(seed, kind, dist.value, dist.min, dist.max, C.c_void_p(ids.data_ptr()), R,
                                     n_roll, C.c_void_p(counts.data_ptr()), C.c_void_p(s)))
    off = torch.zeros(S + 1, dtype=torch.int64, device=dev)
    if S:
        torch.cumsum(counts[:S].to(torch.int64) * bytes_per_token, 0, out=off[1:])
    total = int(off[-1].item())
    payload = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    if total:
        _abi.check(L.dfx_generate_payload(seed, C.c_void_p(ids.data_ptr()), R, n_roll, C.c_void_p(off.data_ptr()),
                                          C.c_void_p(payload.data_ptr()), C.c_void_p(s)))
    return counts[:S].view(torch.uint32) if hasattr(torch, "uint32") else counts[:S], off, payload[:total]
