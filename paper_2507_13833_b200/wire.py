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
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _abi.check(L.dfx_serialize_records(C.byref(st), _ptr(batch.ids), _ptr(tok_count), len(streams),
                                       C.cast(sptr, C.c_void_p), C.cast(esz, C.c_void_p), len(names),
                                       C.cast(cnames, C.c_void_p), C.cast(cptr, C.c_void_p), _ptr(d_meta),
                                       _ptr(d_moff), _ptr(d_rec_off), _ptr(out), s))
    out._keep = (d_rec_off, d_meta, d_moff)
    return out
