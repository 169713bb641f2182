"""Device record serializer (paper_2507_13833_b200/wire.py, csrc/blob.cu) vs the reference wire format.

CPU: dfx_serialize_plan sizes == the oracle serializer's blob lengths (record.hpp:109-127, 187-201).
GPU: device blobs byte-identical to the oracle serializer (pinned to the reference: golden blob of
tests/golden/blobs.npz, and live against the reference compiled into oracle/_ref), over odd-sized streams (u8
mask), empty rollouts, per-record meta sections, views and a reshard's destination groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STREAMS = ("token_id", "lp", "old_lp", "ref_lp", "mask")


def _meta(n, seed):
    """Per-record meta sections (u32 count + (str, str)*), like rec.meta["prompt"] (data_plane.hpp:72)."""
    rng = np.random.default_rng(seed)
    blob, off = bytearray(), [0]
    for r in range(n):
        k = int(rng.integers(0, 3))
        sec = bytearray(int(k).to_bytes(4, "little"))
        for j in range(k):
            key, val = f"k{j}".encode(), bytes(rng.integers(97, 123, int(rng.integers(0, 23))).astype(np.uint8))
            sec += len(key).to_bytes(4, "little") + key + len(val).to_bytes(4, "little") + val
        blob += sec
        off.append(len(blob))
    return np.frombuffer(bytes(blob), np.uint8).copy(), np.array(off, np.int64)


def _host(O, seed, R, n, lo, hi):
    return O.SynthBatch(seed, R, n, O.token_dist("uniform", lo, lo, hi), streams=STREAMS)


@pytest.mark.parametrize("seed,R,n,lo,hi,meta", [(7, 16, 2, 16, 48, False), (3, 33, 5, 0, 37, True),
                                                  (5, 4, 1, 0, 0, True)])
def test_serialize_plan_sizes(O, dfx, seed, R, n, lo, hi, meta):
    from paper_2507_13833_b200 import _abi, wire
    L = wire._declare()
    sb = _host(O, seed, R, n, lo, hi)
    T = sb.n_tokens
    mb, mo = _meta(R, seed) if meta else (None, None)
    blob = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, [getattr(sb, k)[:T] for k in STREAMS],
                              {"advantage": sb.reward, "reward": sb.reward}, meta_off=mo, meta_blob=mb)
    esz = (C.c_uint32 * 5)(4, 4, 4, 4, 1)
    names = (C.c_char_p * 2)(b"advantage", b"reward")
    rec_off = np.zeros(R + 1, np.int64)
    go, cu = np.ascontiguousarray(sb.group_off, np.int32), np.ascontiguousarray(sb.cu_seqlens, np.int64)
    total = L.dfx_serialize_plan(R, go.ctypes.data, cu.ctypes.data, None if mo is None else mo.ctypes.data, 5,
                                 C.cast(esz, C.c_void_p), 2, C.cast(names, C.c_void_p), rec_off.ctypes.data)
    assert total == len(blob)
    assert rec_off[0] == 0 and rec_off[-1] == len(blob) - 4


def _device(dfx, sb):
    T = sb.n_tokens
    return dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward, "value": sb.value},
                                     {k: getattr(sb, k)[:T] for k in STREAMS})


@pytest.mark.gpu
def test_device_blob_matches_golden(O, dfx):
    """The golden blob of tests/golden/blobs.npz (written by the compiled reference)."""
    from paper_2507_13833_b200 import wire
    g = np.load(os.path.join(ROOT, "tests", "golden", "blobs.npz"))
    sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48), streams=STREAMS)
    b = _device(dfx, sb)
    dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, dfx.StageContext())
    out = wire.serialize(b, streams=("token_id", "lp", "old_lp", "ref_lp"), channels=("reward", "advantage"))
    assert out.cpu().numpy().tobytes() == g["blob"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed,R,n,lo,hi,meta,view", [(3, 33, 5, 0, 37, True, None), (11, 64, 8, 1, 700, False, None),
                                                       (5, 20, 3, 0, 9, True, (4, 17)), (9, 3, 1, 0, 0, False, None)])
def test_device_blob_matches_reference(O, dfx, seed, R, n, lo, hi, meta, view):
    from paper_2507_13833_b200 import wire
    sb = _host(O, seed, R, n, lo, hi)
    T = sb.n_tokens
    b = _device(dfx, sb)
    mb, mo = _meta(R, seed) if meta else (None, None)
    ids, go, cu, tc = sb.ids, sb.group_off, sb.cu_seqlens, sb.tok_count
    rew, val = sb.reward, sb.value
    if view is not None:  # records [r0, r1): a zero-copy view with token_base > 0
        r0, r1 = view
        b = b.view_records(r0, r1)
        s0, s1 = int(go[r0]), int(go[r1])
        ids, tc, rew, val = ids[r0:r1], tc[s0:s1], rew[s0:s1], val[s0:s1]
        cu = np.ascontiguousarray(cu[s0:s1 + 1])
        go = (go[r0:r1 + 1] - s0).astype(np.int32)
        if meta:
            mb = mb[mo[r0]:mo[r1]].copy()
            mo = (mo[r0:r1 + 1] - mo[r0]).astype(np.int64)
    out = wire.serialize(b, streams=STREAMS, channels=("reward", "value"), meta_blob=mb, meta_off=mo)
    want = O.serialize_packed(ids, go, tc, cu, [getattr(sb, k)[:T] for k in STREAMS], {"reward": rew, "value": val},
                              meta_off=mo, meta_blob=mb)
    assert out.cpu().numpy().tobytes() == want.tobytes()
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdistflow_ref.so")):
        ref = O.serialize_packed(ids, go, tc, cu, [getattr(sb, k)[:T] for k in STREAMS], {"reward": rew, "value": val},
                                 meta_off=mo, meta_blob=mb, use_reference=True)
        assert want.tobytes() == ref.tobytes()


def test_blob_index_rejects_malformed(O, dfx):
    """Header walk on the CPU: truncation and channel-set mismatches raise (the reference's ParseError)."""
    from paper_2507_13833_b200 import errors, wire
    sb = _host(O, 7, 6, 2, 1, 20)
    T = sb.n_tokens
    blob = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, [getattr(sb, k)[:T] for k in STREAMS],
                              {"advantage": sb.reward, "reward": sb.reward})
    with pytest.raises(errors.Error):
        wire.deserialize(blob[:-3], device="cpu")
    with pytest.raises(errors.Error):
        wire.deserialize(blob, channels=("reward",), device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("seed,R,n,lo,hi,meta", [(3, 33, 5, 0, 37, True), (7, 16, 2, 16, 48, False)])
def test_blob_round_trip(O, dfx, seed, R, n, lo, hi, meta):
    """reference bytes -> device batch (dfx_blob_index + dfx_blob_unpack) -> device bytes: identical, and the
    device streams / channels equal the records' values bit for bit."""
    from paper_2507_13833_b200 import wire
    sb = _host(O, seed, R, n, lo, hi)
    T = sb.n_tokens
    mb, mo = _meta(R, seed) if meta else (None, None)
    blob = O.serialize_packed(sb.ids, sb.group_off, sb.tok_count, sb.cu_seqlens, [getattr(sb, k)[:T] for k in STREAMS],
                              {"advantage": sb.value, "reward": sb.reward}, meta_off=mo, meta_blob=mb)
    b, (meta_blob, meta_off, tc) = wire.deserialize(blob)
    assert tc.tolist() == sb.tok_count.tolist()
    for k in STREAMS:
        assert b.streams[k][:T].cpu().numpy().tobytes() == getattr(sb, k)[:T].tobytes(), k
    assert b.channels["reward"].cpu().numpy().tobytes() == sb.reward.tobytes()
    assert b.channels["advantage"].cpu().numpy().tobytes() == sb.value.tobytes()
    if meta:
        assert meta_blob.tobytes() == mb.tobytes() and meta_off.tolist() == mo.tolist()
    again = wire.serialize(b, channels=("advantage", "reward"), meta_blob=meta_blob if meta else None,
                           meta_off=meta_off if meta else None)
    assert again.cpu().numpy().tobytes() == blob.tobytes()
