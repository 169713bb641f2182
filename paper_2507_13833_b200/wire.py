"""The reference's record wire format from device batches.

serialize(batch, ...) writes serialize_records (distflow/record.hpp:109-127, 151-156) of a device PackedBatch on
the GPU (dfx_serialize_records): the blob a CPU peer (Fabric / BufferStore::exchange) reads, byte-identical to the
reference serializer, without packing records on the host first.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi, errors
from .packed import PackedBatch, _ptr

PAYLOAD_STREAMS = ("token_id", "lp", "old_lp", "ref_lp", "mask")  # DESIGN.md §3 payload layout (17 B/token)


def _declare():
    L = _abi.lib()
    if getattr(L, "_wire_declared", False):
        return L
    P = C.c_void_p
    L.dfx_serialize_plan.restype = C.c_int64
    L.dfx_serialize_plan.argtypes = [C.c_int64, P, P, P, C.c_int32, P, C.c_int32, P, P]
    L.dfx_serialize_records.restype = C.c_int32
    L.dfx_serialize_records.argtypes = [C.POINTER(_abi.Packed), P, P, C.c_int32, P, P, C.c_int32, P, P, P, P, P, P, P]
    L._wire_declared = True
    return L


def serialize(batch: PackedBatch, streams=PAYLOAD_STREAMS, channels=None, meta_blob: np.ndarray | None = None,
              meta_off: np.ndarray | None = None, tok_count: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device blob (uint8 tensor) of the batch's records. channels: names to write (default: all rollout
    channels, sorted like std::map); meta_blob/meta_off: per-record pre-serialized meta sections (host)."""
    run, out = serialize_prepared(batch, streams, channels, meta_blob, meta_off, tok_count)
    run(out, stream)
    return out


def serialize_prepared(batch: PackedBatch, streams=PAYLOAD_STREAMS, channels=None, meta_blob=None, meta_off=None,
                       tok_count=None):
    """The host plan and device arguments of serialize(), once: returns (run, out) where run(out, stream=None)
    launches only the device serializer into `out` (repeatable; e.g. for timing the kernel alone)."""
    L = _declare()
    batch.ensure_host_meta()
    dev = batch.device
    names = sorted(batch.channels if channels is None else channels)
    for n in names:
        if n not in batch.channels:
            raise errors.MissingChannelError(n)
    for k in streams:
        if k not in batch.streams:
            raise errors.MissingChannelError(k)
    esz = (C.c_uint32 * max(1, len(streams)))(*[batch.streams[k].element_size() for k in streams])
    cnames = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    R = batch.n_records
    rec_off = np.zeros(R + 1, np.int64)
    hgo = np.ascontiguousarray(batch.host_group_off, np.int32)
    hcu = np.ascontiguousarray(batch.host_cu, np.int64)
    hmo = None if meta_off is None else np.ascontiguousarray(meta_off, np.int64)
    total = L.dfx_serialize_plan(R, hgo.ctypes.data, hcu.ctypes.data, None if hmo is None else hmo.ctypes.data,
                                 len(streams), C.cast(esz, C.c_void_p), len(names), C.cast(cnames, C.c_void_p),
                                 rec_off.ctypes.data)
    if total < 0:
        _abi.check(int(-total))
    out = torch.empty(int(total), dtype=torch.uint8, device=dev)
    d_rec_off = torch.from_numpy(rec_off).to(dev)
    d_meta = d_moff = None
    if meta_blob is not None:
        d_meta = torch.zeros(len(meta_blob) + 8, dtype=torch.uint8, device=dev)  # 4+ bytes of read slack
        d_meta[: len(meta_blob)].copy_(torch.from_numpy(np.ascontiguousarray(meta_blob, np.uint8)))
        d_moff = torch.from_numpy(hmo).to(dev)
    sptr = (C.c_void_p * max(1, len(streams)))(*[batch.streams[k].data_ptr() for k in streams])
    cptr = (C.c_void_p * max(1, len(names)))(*[batch.channels[n].data_ptr() for n in names])
    st = batch.struct()
    out._keep = (d_rec_off, d_meta, d_moff)

    def run(dst, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _abi.check(L.dfx_serialize_records(C.byref(st), _ptr(batch.ids), _ptr(tok_count), len(streams),
                                           C.cast(sptr, C.c_void_p), C.cast(esz, C.c_void_p), len(names),
                                           C.cast(cnames, C.c_void_p), C.cast(cptr, C.c_void_p), _ptr(d_meta),
                                           _ptr(d_moff), _ptr(d_rec_off), _ptr(dst), s))
    return run, out


def deserialize(blob: np.ndarray, streams=(("token_id", torch.int32), ("lp", torch.float32), ("old_lp", torch.float32),
                                          ("ref_lp", torch.float32), ("mask", torch.uint8)),
                channels=("advantage", "reward"), device="cuda", stream=None):
    """A record blob (host bytes, e.g. from a CPU Fabric peer) -> device PackedBatch: host header walk
    (dfx_blob_index), then one H2D of the blob and a device gather of payloads and channels (dfx_blob_unpack).
    Returns (batch, (meta_blob, meta_off, tok_count)): the per-record meta sections gathered contiguously (host),
    ready for serialize(..., meta_blob=, meta_off=)."""
    L = _abi.lib()
    P = C.c_void_p
    L.dfx_blob_index.argtypes = [P, C.c_uint64, C.c_uint32, C.c_int32, P] + [P] * 10
    L.dfx_blob_unpack.argtypes = [P, C.c_int64, P, P, P, C.c_int32, P, P, C.c_int32, P, P, P]
    blob = np.ascontiguousarray(blob, np.uint8)
    names = list(channels)
    cn = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    esz = [torch.empty(0, dtype=dt).element_size() for _, dt in streams]
    bpt = sum(esz)
    nr, ns, nt = C.c_int64(), C.c_int64(), C.c_int64()
    args = (blob.ctypes.data, blob.size, bpt, len(names), C.cast(cn, C.c_void_p), C.byref(nr), C.byref(ns), C.byref(nt))
    _abi.check(L.dfx_blob_index(*args, *([None] * 7)))
    R, S, T = nr.value, ns.value, nt.value
    ids = np.zeros(R, np.uint64)
    meta_range = np.zeros(2 * max(R, 1), np.int64)
    go = np.zeros(R + 1, np.int32)
    cu = np.zeros(S + 1, np.int64)
    tc = np.zeros(max(S, 1), np.uint32)
    po = np.zeros(max(S, 1), np.int64)
    co = np.zeros(max(S, 1), np.int64)
    _abi.check(L.dfx_blob_index(*args, ids.ctypes.data, meta_range.ctypes.data, go.ctypes.data, cu.ctypes.data,
                                tc.ctypes.data, po.ctypes.data, co.ctypes.data))
    from .packed import padded_len
    b = PackedBatch.from_host(ids, go, cu, {}, None, device=device)
    dev = b.device
    d_blob = torch.empty(blob.size + 8, dtype=torch.uint8, device=dev)
    d_blob[: blob.size].copy_(torch.from_numpy(blob))
    d_po = torch.from_numpy(po).to(dev)
    d_co = torch.from_numpy(co).to(dev)
    outs = {n: torch.zeros(padded_len(T), dtype=dt, device=dev) for n, dt in streams}
    chs = {n: torch.empty(S, dtype=torch.float64, device=dev) for n in names}
    sp = (C.c_void_p * max(1, len(streams)))(*[outs[n].data_ptr() for n, _ in streams])
    ez = (C.c_uint32 * max(1, len(streams)))(*esz)
    cp = (C.c_void_p * max(1, len(names)))(*[chs[n].data_ptr() for n in names])
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _abi.check(L.dfx_blob_unpack(d_blob.data_ptr(), S, b.cu_seqlens.data_ptr(), d_po.data_ptr(), d_co.data_ptr(),
                                 len(streams), C.cast(sp, C.c_void_p), C.cast(ez, C.c_void_p), len(names),
                                 C.cast(cn, C.c_void_p), C.cast(cp, C.c_void_p), s))
    b.streams.update(outs)
    b.channels.update(chs)
    b._keep_blob = (d_blob, d_po, d_co)
    sec = [blob[meta_range[2 * r]:meta_range[2 * r + 1]] for r in range(R)]
    meta_off = np.zeros(R + 1, np.int64)
    np.cumsum([len(x) for x in sec], out=meta_off[1:])
    meta_blob = np.concatenate(sec) if sec else np.zeros(0, np.uint8)
    return b, (meta_blob, meta_off, tc[:S])
