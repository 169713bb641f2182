"""NativeBufferStore: the reference BufferStore (distflow/data_plane.hpp:225-457) for one process per GPU, run by
libdfx's distributed DataBuffer (csrc/dstore.cu, include/dfx.h "Distributed DataBuffer").

Every verb is ONE call into the C ABI -- the host metadata exchange (shared memory between the box's processes),
the placement, the remote transfers (copy-engine pulls of peer-mapped producer memory over NVLink, or NCCL
send/recv), the local copies and the metadata unpack all happen natively on the caller's stream; Python only
marshals pointers. Same verbs, semantics and error types as the reference:
  put            TP != 0 suppressed (:245-248), group must be local, duplicates / stale iterations raise
  ensure_ready   collective over the communicator (every rank calls it for the same stage / iteration, like the
                 reference's SPMD exchange, :296-346, :400-442); NotReadyError when a local put is missing
  get            the destination group's batch on this GPU (TP peers on one GPU share it, :269-292); its device
                 memory belongs to the store until worker_done retires the iteration
  worker_done    once per local logical worker (:351-367)

Communicator: Comm.create(world, rank) -- rank 0 makes the NCCL id, torch.distributed (any backend) only carries
its 128 bytes once at setup; no torch collective is used on the data path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi, errors
from .packed import PackedBatch
from .reshard import Layout, Topology

P = C.c_void_p
MAX_CH, MAX_STREAMS, ID_BYTES = 4, 8, 128


class Batch(C.Structure):
    """dfx_batch (include/dfx.h)."""
    _fields_ = [("n_records", C.c_int64), ("n_rollouts", C.c_int64), ("token_base", C.c_int64),
                ("token_span", C.c_int64), ("ids", P), ("group_off", P), ("roll_group", P), ("cu_seqlens", P),
                ("ch", P * MAX_CH), ("st", P * MAX_STREAMS), ("h_group_off", P), ("h_cu", P)]


class StoreCfg(C.Structure):
    """dfx_dstore_cfg (include/dfx.h)."""
    _fields_ = [("num_nodes", C.c_uint32), ("workers_per_node", C.c_uint32), ("rank_of_worker", P),
                ("n_streams", C.c_int32), ("stream_esz", P), ("n_ch", C.c_int32), ("n_stages", C.c_int32),
                ("stage_names", P), ("produced_dp", P), ("produced_tp", P), ("consumed_dp", P), ("consumed_tp", P),
                ("transport", C.c_int32)]


def _declare():
    L = _abi.lib()
    if getattr(L, "_dstore_declared", False):
        return L
    st = C.c_int32
    L.dfx_comm_unique_id.argtypes = [P]
    L.dfx_comm_unique_id.restype = st
    L.dfx_comm_init.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(P)]
    L.dfx_comm_init.restype = st
    L.dfx_comm_destroy.argtypes = [P]
    L.dfx_comm_destroy.restype = st
    L.dfx_comm_allreduce_i64.argtypes = [P, P, P, C.c_int64, P]
    L.dfx_comm_allreduce_i64.restype = st
    L.dfx_dstore_create.argtypes = [C.POINTER(StoreCfg), P, P, C.POINTER(P)]
    L.dfx_dstore_create.restype = st
    L.dfx_dstore_destroy.argtypes = [P]
    L.dfx_dstore_destroy.restype = st
    L.dfx_dstore_put.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(Batch),
                                 C.POINTER(C.c_int32)]
    L.dfx_dstore_put.restype = st
    L.dfx_dstore_ensure_ready.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32]
    L.dfx_dstore_ensure_ready.restype = st
    L.dfx_dstore_get.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(Batch)]
    L.dfx_dstore_get.restype = st
    L.dfx_dstore_worker_done.argtypes = [P, C.c_uint64]
    L.dfx_dstore_worker_done.restype = st
    L.dfx_dstore_stats.argtypes = [P, P]
    L.dfx_dstore_stats.restype = st
    L._dstore_declared = True
    return L


class Comm:
    """An NCCL communicator of libdfx over the participating GPUs (one rank per process, current device)."""

    def __init__(self, handle: int, world: int, rank: int):
        self.handle, self.world, self.rank = handle, world, rank

    @staticmethod
    def create(world: int, rank: int, group=None) -> "Comm":
        L = _declare()
        buf = (C.c_char * ID_BYTES)()
        if rank == 0:
            _abi.check(L.dfx_comm_unique_id(buf))
        if world > 1:  # setup only: ship rank 0's id bytes
            import torch.distributed as dist
            obj = [bytes(buf) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(buf, obj[0], ID_BYTES)
        h = P()
        _abi.check(L.dfx_comm_init(buf, world, rank, C.byref(h)))
        return Comm(h.value, world, rank)

    def allreduce_i64(self, values, stream=None) -> np.ndarray:
        a = np.ascontiguousarray(values, np.int64)
        out = np.zeros_like(a)
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _abi.check(_declare().dfx_comm_allreduce_i64(self.handle, a.ctypes.data, out.ctypes.data, a.size, st))
        return out

    def close(self):
        if self.handle:
            _declare().dfx_comm_destroy(self.handle)
            self.handle = None


class _CudaArray:
    """__cuda_array_interface__ over store-owned device memory (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, n: int, typestr: str, dev: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}
        self.dev = dev


_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1"}


def _wrap(ptr, n, dtype, dev) -> torch.Tensor:
    if n == 0 or not ptr:
        return torch.empty(0, dtype=dtype, device=dev)
    return torch.as_tensor(_CudaArray(ptr, n, _TYPESTR[dtype], dev.index), device=dev)


class NativeBufferStore:
    """See the module docstring. streams: [(name, torch dtype)] and channels: [name] fix the schema of the batches
    (every put batch carries them). stages: {name: StoreStagePlan}."""

    def __init__(self, topo: Topology, comm: Comm, stages: dict, streams, channels, stream=None,
                 transport: str = "pull"):
        L = _declare()
        self.topo, self.comm = topo, comm
        self.stream_specs = [(n, dt) for n, dt in streams]
        self.ch_names = list(channels)
        if len(self.stream_specs) > MAX_STREAMS or len(self.ch_names) > MAX_CH:
            raise errors.Error("too many streams or channels for the native store")
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self.local_workers = [w for w in range(topo.world) if topo.gpu_of_worker[w] == comm.rank]
        names = list(stages)
        self._keep = [np.array(topo.gpu_of_worker, np.int32),
                      np.array([torch.empty(0, dtype=dt).element_size() for _, dt in self.stream_specs], np.uint32),
                      (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names]),
                      np.array([stages[n].produced.dp for n in names], np.uint32),
                      np.array([stages[n].produced.tp for n in names], np.uint32),
                      np.array([stages[n].consumed.dp if stages[n].consumed else 0 for n in names], np.uint32),
                      np.array([stages[n].consumed.tp if stages[n].consumed else 0 for n in names], np.uint32)]
        k = self._keep
        cfg = StoreCfg(topo.num_nodes, topo.workers_per_node, k[0].ctypes.data, len(self.stream_specs),
                       k[1].ctypes.data, len(self.ch_names), len(names), C.cast(k[2], P), k[3].ctypes.data,
                       k[4].ctypes.data, k[5].ctypes.data, k[6].ctypes.data, {"pull": 0, "nccl": 1}[transport])
        h = P()
        _abi.check(L.dfx_dstore_create(C.byref(cfg), comm.handle, self.stream.cuda_stream, C.byref(h)))
        self.handle = h.value
        self._puts = {}  # (stage, iteration) -> batches kept alive until the exchange has read them
        self._wrapped = {}  # (stage, dest group) -> tensors over the store's memory, reused while it is the same
        self._L = L

    def close(self):
        if self.handle:
            _declare().dfx_dstore_destroy(self.handle)
            self.handle = None

    # ---- verbs ---------------------------------------------------------------------------------
    def _batch_struct(self, b: PackedBatch):
        """The dfx_batch of a PackedBatch, cached on the batch while its arrays stay the same (a training loop
        re-puts the same buffers every iteration)."""
        b.ensure_host_meta()
        b._materialize()
        chs = [b.channels.get(n) for n in self.ch_names]
        sts = [b.streams.get(n) for n, _ in self.stream_specs]
        for n, t in zip(self.ch_names + [n for n, _ in self.stream_specs], chs + sts):
            if t is None:
                raise errors.MissingChannelError(n)
        key = (b.n_records, b.n_rollouts, b.token_base, b.token_span, b.ids.data_ptr(), b.group_off.data_ptr(),
               b.roll_group.data_ptr(), b.cu_seqlens.data_ptr(), id(b.host_group_off), id(b.host_cu),
               *[t.data_ptr() for t in chs], *[t.data_ptr() for t in sts])
        cached = getattr(b, "_dstore_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1], cached[2]
        s = Batch()
        s.n_records, s.n_rollouts, s.token_base, s.token_span = b.n_records, b.n_rollouts, b.token_base, b.token_span
        s.ids, s.group_off, s.roll_group, s.cu_seqlens = key[4:8]
        for c, t in enumerate(chs):
            s.ch[c] = t.data_ptr()
        for k, t in enumerate(sts):
            s.st[k] = t.data_ptr()
        go = np.ascontiguousarray(b.host_group_off, np.int32)
        cu = np.ascontiguousarray(b.host_cu, np.int64)
        s.h_group_off, s.h_cu = go.ctypes.data, cu.ctypes.data
        b._dstore_cache = (key, s, (go, cu))
        return s, (go, cu)

    def batch_struct(self, b: PackedBatch) -> Batch:
        """The dfx_batch of a PackedBatch (for put_raw); valid while the batch is alive and unchanged."""
        return self._batch_struct(b)[0]

    def put(self, stage: str, iteration: int, dp_rank: int, tp_rank: int, batch: PackedBatch) -> bool:
        s, keep = self._batch_struct(batch)
        acc = C.c_int32()
        _abi.check(_declare().dfx_dstore_put(self.handle, stage.encode(), iteration, dp_rank, tp_rank, C.byref(s),
                                             C.byref(acc)))
        if acc.value:
            self._puts.setdefault((stage, iteration), []).append((batch, keep))
        return bool(acc.value)

    def ensure_ready(self, stage: str, iteration: int, to: Layout) -> None:
        _abi.check(_declare().dfx_dstore_ensure_ready(self.handle, stage.encode(), iteration, to.dp, to.tp))

    def get(self, stage: str, iteration: int, dest_dp: int, to: Layout) -> PackedBatch:
        """The destination group's batch as a PackedBatch over store-owned memory (no copy), valid until
        worker_done(iteration) has been called by every local worker. The tensors wrapping the store's memory are
        reused while the store hands out the same buffers (its block cache does, in a steady-state loop)."""
        b = Batch()
        _abi.check(_declare().dfx_dstore_get(self.handle, stage.encode(), iteration, dest_dp, to.dp, to.tp,
                                             C.byref(b)))
        R, S, T0, T = b.n_records, b.n_rollouts, b.token_base, b.token_span
        dev = self.dev
        hgo = np.ctypeslib.as_array(C.cast(b.h_group_off, C.POINTER(C.c_int32)), (R + 1,)).copy()
        hcu = np.ctypeslib.as_array(C.cast(b.h_cu, C.POINTER(C.c_int64)), (S + 1,)).copy()
        n_tok = T0 + T + 16  # the streams are addressed from token 0 of their coordinate system (+ over-read slack)
        key = (R, S, T0, T, b.ids, b.group_off, b.roll_group, b.cu_seqlens, *b.ch[:len(self.ch_names)],
               *b.st[:len(self.stream_specs)])
        wrapped = self._wrapped.get((stage, dest_dp))
        if wrapped is None or wrapped[0] != key:
            wrapped = (key, (_wrap(b.ids, R, torch.int64, dev), _wrap(b.group_off, R + 1, torch.int32, dev),
                             _wrap(b.roll_group, S, torch.int32, dev), _wrap(b.cu_seqlens, S + 1, torch.int64, dev),
                             {n: _wrap(b.ch[c], S, torch.float64, dev) for c, n in enumerate(self.ch_names)},
                             {n: _wrap(b.st[k], n_tok, dt, dev) for k, (n, dt) in enumerate(self.stream_specs)}))
            self._wrapped[(stage, dest_dp)] = wrapped
        ids, go, rg, cu, chs, sts = wrapped[1]
        return PackedBatch(R, S, T0, T, ids, go, rg, cu, dict(chs), dict(sts), host_group_off=hgo, host_cu=hcu)

    # ---- raw verbs: the C structs straight through (a consumer group re-put into the next stage needs no tensors;
    # this is what a C++ caller does, include/dfx_dstore.hpp) ----
    def put_raw(self, stage: bytes, iteration: int, dp_rank: int, tp_rank: int, s: Batch) -> bool:
        acc = C.c_int32()
        _abi.check(self._L.dfx_dstore_put(self.handle, stage, iteration, dp_rank, tp_rank, C.byref(s), C.byref(acc)))
        return bool(acc.value)

    def get_raw(self, stage: bytes, iteration: int, dest_dp: int, to: Layout, out: Batch) -> Batch:
        _abi.check(self._L.dfx_dstore_get(self.handle, stage, iteration, dest_dp, to.dp, to.tp, C.byref(out)))
        return out

    def ensure_ready_raw(self, stage: bytes, iteration: int, to: Layout) -> None:
        _abi.check(self._L.dfx_dstore_ensure_ready(self.handle, stage, iteration, to.dp, to.tp))

    def worker_done_raw(self, iteration: int) -> None:
        _abi.check(self._L.dfx_dstore_worker_done(self.handle, iteration))

    def worker_done(self, iteration: int) -> None:
        _abi.check(_declare().dfx_dstore_worker_done(self.handle, iteration))
        for k in [k for k in self._puts if k[1] <= iteration]:
            del self._puts[k]

    def stats(self) -> dict:
        out = np.zeros(5, np.uint64)
        _abi.check(_declare().dfx_dstore_stats(self.handle, out.ctypes.data))
        return dict(zip(("suppressed", "bytes_sent", "bytes_recv", "bytes_copied", "plan_hits"), out.tolist()))
