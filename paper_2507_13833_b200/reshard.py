"""DataBuffer DP m->n reshard of device-resident packed batches.

Replaces BufferStore::exchange/get (distflow/data_plane.hpp:296-442) and all_to_all (distflow/transport.hpp:718-754)
for the GPU path. The reference placement is computed natively (dfx_reshard_segments, csrc/reshard.cu) as segments:
runs of consecutive records of one producer group that land consecutively in one consumer group. Logical workers
(the reference's B x W ranks) are mapped onto GPUs (one process per GPU); a producer group lives on the GPU of
its TP-0 worker (only TP-0 puts, data_plane.hpp:245-248) and a consumer group is needed on every GPU hosting one
of its TP workers (TP peers read identical batches, :266-292).

Per exchange, on every rank (SPMD, all ranks call it for the same stage/iteration like ensure_ready):
  1. sizes: rollout/token counts of every segment, filled by the owning rank from its host metadata and summed
     over ranks (one small all-reduce; skipped on a single GPU);
  2. a consumer batch holding this rank's consumer groups in dp order -- a zero-copy view when all of them are one
     contiguous run of a local producer batch (every box placement with <= 4 GPUs), else freshly allocated;
  3. token streams move as contiguous byte ranges: device copies when local, NCCL send/recv (grouped, one
     ncclGroupStart/End) across GPUs over NVLink; record/rollout metadata moves as one packed buffer per
     segment (dfx_reshard_pack) and is rebased into the consumer batch by dfx_reshard_unpack.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, errors
from .packed import PackedBatch, padded_len

CHANNELS = ("reward", "value", "advantage")

# debug instrumentation (tools/prof_exchange.py): phase -> accumulated seconds, synchronised per phase
PROFILE = None


def _mark(name, t0):
    if PROFILE is None:
        return None
    import time
    torch.cuda.synchronize()
    t = time.perf_counter()
    if t0 is not None:
        PROFILE[name] = PROFILE.get(name, 0.0) + t - t0
    return t


class Segment(C.Structure):
    _fields_ = [("dst_group", C.c_uint32), ("src_group", C.c_uint32), ("dst_rec", C.c_uint64),
                ("src_rec", C.c_uint64), ("count", C.c_uint64)]


class SegMeta(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("group_off", C.c_void_p), ("cu", C.c_void_p), ("ch", C.c_void_p * 4),
                ("n_rec", C.c_int64), ("n_roll", C.c_int64), ("dst_rec", C.c_int64), ("dst_roll", C.c_int64),
                ("dst_tok", C.c_int64)]


def _declare():
    L = _abi.lib()
    if getattr(L, "_reshard_declared", False):
        return L
    P = C.c_void_p
    L.dfx_reshard_placement.argtypes = [C.c_uint32] * 6 + [P, P, P]
    L.dfx_reshard_placement.restype = C.c_int32
    L.dfx_reshard_segments.argtypes = [C.c_uint32] * 6 + [P, P, C.c_int64]
    L.dfx_reshard_segments.restype = C.c_int64
    L.dfx_reshard_pack_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int32]
    L.dfx_reshard_pack_bytes.restype = C.c_int64
    L.dfx_reshard_pack.argtypes = [P, C.c_int32, C.c_int32, P, P]
    L.dfx_reshard_pack.restype = C.c_int32
    L.dfx_reshard_unpack.argtypes = [P, C.c_int32, C.c_int32, P, P, P, P, P, P]
    L.dfx_reshard_unpack.restype = C.c_int32
    L.dfx_ipc_export.argtypes = [P, P, C.POINTER(C.c_uint64)]
    L.dfx_ipc_export.restype = C.c_int32
    L.dfx_ipc_open.argtypes = [P, C.c_size_t, C.POINTER(C.c_void_p)]
    L.dfx_ipc_open.restype = C.c_int32
    L.dfx_ipc_close.argtypes = [P]
    L.dfx_ipc_close.restype = C.c_int32
    L.dfx_ipc_open_count.argtypes = []
    L.dfx_ipc_open_count.restype = C.c_int64
    L.dfx_copy_async.argtypes = [P, P, C.c_size_t, P]
    L.dfx_copy_batch.argtypes = [C.c_int64, P, P, P, P]
    L.dfx_copy_batch.restype = C.c_int32
    L.dfx_copy_many.argtypes = [C.c_int64, P, P, P, P]
    L.dfx_copy_many.restype = C.c_int32
    L.dfx_copy_async.restype = C.c_int32
    L._reshard_declared = True
    return L


@dataclass(frozen=True)
class Layout:
    """distflow::ParallelLayout (topology.hpp:40-51)."""
    dp: int
    tp: int

    def dp_rank(self, w: int) -> int:
        return w // self.tp

    def tp_rank(self, w: int) -> int:
        return w % self.tp

    def group_lead(self, d: int) -> int:
        return d * self.tp


@dataclass(frozen=True)
class Topology:
    """distflow::ClusterTopology (topology.hpp:11-35) plus the logical-worker -> GPU (process rank) mapping."""
    num_nodes: int
    workers_per_node: int
    gpu_of_worker: tuple

    @property
    def world(self) -> int:
        return self.num_nodes * self.workers_per_node

    @staticmethod
    def box(workers: int, n_gpus: int) -> "Topology":
        """One DataBuffer per box (B = 1), W logical workers spread evenly over the GPUs."""
        if workers % n_gpus:
            raise errors.LayoutError(f"{workers} logical workers cannot be spread over {n_gpus} GPUs")
        return Topology(1, workers, tuple(w // (workers // n_gpus) for w in range(workers)))

    @staticmethod
    def store_per_gpu(n_gpus: int, workers_per_gpu: int) -> "Topology":
        """One DataBuffer per GPU (B = n_gpus, W = workers_per_gpu)."""
        return Topology(n_gpus, workers_per_gpu,
                        tuple(w // workers_per_gpu for w in range(n_gpus * workers_per_gpu)))


def placement(topo: Topology, produced: Layout, consumed: Layout, group_counts):
    """The reference's record placement: (dest_counts, src_index) -- see dfx_reshard_placement."""
    L = _declare()
    gc = np.ascontiguousarray(group_counts, np.uint64)
    dc = np.zeros(consumed.dp, np.uint64)
    idx = np.zeros(max(int(gc.sum()), 1), np.uint64)
    _abi.check(L.dfx_reshard_placement(topo.num_nodes, topo.workers_per_node, produced.dp, produced.tp, consumed.dp,
                                       consumed.tp, gc.ctypes.data, dc.ctypes.data, idx.ctypes.data))
    return dc, idx[: int(gc.sum())]


def segments(topo: Topology, produced: Layout, consumed: Layout, group_counts) -> list:
    L = _declare()
    gc = np.ascontiguousarray(group_counts, np.uint64)
    args = (topo.num_nodes, topo.workers_per_node, produced.dp, produced.tp, consumed.dp, consumed.tp, gc.ctypes.data)
    n = L.dfx_reshard_segments(*args, None, 0)
    if n < 0:
        _abi.check(int(-n))
    buf = (Segment * max(n, 1))()
    L.dfx_reshard_segments(*args, C.cast(buf, C.c_void_p), n)
    return [(s.dst_group, s.src_group, s.dst_rec, s.src_rec, s.count) for s in buf[:n]]


class Plan:
    """Segments plus where every producer / consumer group lives."""

    def __init__(self, topo: Topology, produced: Layout, consumed: Layout, group_counts, rank: int):
        if len(topo.gpu_of_worker) != topo.world:
            raise errors.LayoutError("gpu_of_worker must map every logical worker")
        self.topo, self.produced, self.consumed, self.rank = topo, produced, consumed, rank
        self.group_counts = np.asarray(group_counts, np.uint64)
        self.segs = segments(topo, produced, consumed, group_counts)
        self.src_rank = [topo.gpu_of_worker[produced.group_lead(p)] for p in range(produced.dp)]
        self.dst_ranks = [sorted({topo.gpu_of_worker[consumed.group_lead(d) + t] for t in range(consumed.tp)})
                          for d in range(consumed.dp)]
        self.local_src = [p for p in range(produced.dp) if self.src_rank[p] == rank]
        self.local_dst = [d for d in range(consumed.dp) if rank in self.dst_ranks[d]]
        self.dest_counts = np.zeros(consumed.dp, np.int64)
        for d, p, dr, sr, n in self.segs:
            self.dest_counts[d] += n
        # does any record cross GPUs? (box placements on <= 4 GPUs: never)
        self.cross = any(self.src_rank[p] != r for d, p, _, _, _ in self.segs for r in self.dst_ranks[d])


@dataclass
class RemoteSource:
    """A run of consecutive records of a producer batch held by another GPU, mapped into this GPU's address space
    (CUDA IPC over NVLink): device addresses of the run's first ids / group_off / cu_seqlens / channel entries and
    the base addresses of the token streams (absolute token coordinates, like the producer's own cu_seqlens).
    Kernels read it in place over NVLink; nothing is copied."""
    rank: int
    n_records: int
    n_rollouts: int
    token_base: int
    token_span: int
    addr: dict

    def struct(self) -> _abi.Packed:
        a = self.addr
        return _abi.Packed(self.n_records, self.n_rollouts, a.get("group_off"), None, a.get("cu"), a.get("c:reward"),
                           a.get("c:value"), a.get("s:lp"), a.get("s:old_lp"), a.get("s:ref_lp"), a.get("s:value_tok"),
                           a.get("s:token_reward"), a.get("s:mask"))


@dataclass
class ConsumerBatch:
    """This rank's consumer groups, concatenated in dp order, with per-group record/rollout offsets. A lazy
    exchange (exchange(..., lazy=True)) has batch None and, per group, the token sources in order: local
    PackedBatch views and RemoteSource runs on peer GPUs; release() must follow its last use (device barrier)."""
    batch: PackedBatch | None
    groups: list            # consumer dp ranks held here, in order
    rec_off: list           # record offsets per group (len(groups)+1)
    roll_off: list          # rollout offsets per group
    zero_copy: bool
    bytes_sent: int = 0
    bytes_recv: int = 0
    sources: list | None = None   # lazy: per group, [PackedBatch | RemoteSource]
    release: object = None        # lazy: callable issuing the closing device barrier
    ipc_bases: list | None = None  # peer mappings this exchange opened (dfx_ipc_open); see close_mappings()
    template_owned: bool = False   # a store / exchange template holds this batch's mappings beyond its iteration

    def close_mappings(self) -> None:
        """Drop the references this exchange took on peer mappings (the store calls it when the batch -- or the
        template holding it -- is retired). Every read of them must have completed: the stream is synchronized."""
        if not self.ipc_bases:
            return
        torch.cuda.current_stream().synchronize()
        L = _declare()
        for b in self.ipc_bases:
            _abi.check(L.dfx_ipc_close(C.c_void_p(b)))
        self.ipc_bases = None

    def group_view(self, d: int) -> PackedBatch:
        i = self.groups.index(d)
        if self.rec_off[i] == 0 and self.rec_off[i + 1] == self.batch.n_records:
            return self.batch
        return self.batch.view_records(self.rec_off[i], self.rec_off[i + 1])

    @property
    def loss_group_off(self) -> list:
        return list(self.roll_off)


def _view_consistent(v: PackedBatch) -> bool:
    """A view may be addressed through its parent only if every channel and stream it carries is still the
    parent's storage (a stage function may have attached new channels to the view alone)."""
    par = v.parent
    s0 = int(par.host_group_off[v.parent_rec])
    for c, t in v.channels.items():
        pt = par.channels.get(c)
        if pt is None or t.data_ptr() != pt.data_ptr() + s0 * pt.element_size():
            return False
    return set(v.streams) == set(par.streams) and all(v.streams[k] is par.streams[k] for k in v.streams)


def _src_slices(plan: Plan, sources: dict):
    """Per segment: (src batch, r0, r1, s0, s1, t0, t1) for locally held producer groups (host metadata)."""
    out = {}
    for i, (d, p, dr, sr, n) in enumerate(plan.segs):
        if p not in sources:
            continue
        b, rbase = sources[p]
        if b.parent is not None and _view_consistent(b):  # address the parent so contiguity is visible
            b, rbase = b.parent, b.parent_rec + rbase
        else:
            b._materialize()
        b.ensure_host_meta()
        go, cu = b.host_group_off, b.host_cu
        r0, r1 = rbase + int(sr), rbase + int(sr) + int(n)
        s0, s1 = int(go[r0]), int(go[r1])
        out[i] = (b, r0, r1, s0, s1, int(cu[s0]), int(cu[s1]))
    return out


def exchange(plan: Plan, sources: dict, stream=None, group=None, schema=None, meta_group=None,
             transport: str = "pull", lazy: bool = False, templates: dict | None = None,
             template_key=None) -> ConsumerBatch:
    """Run the reshard on this rank. sources: {producer dp rank: (PackedBatch, first record of that group in it)}
    for every locally held producer group. schema: (stream name -> dtype, channel names), needed only on ranks
    that hold no producer group. Collective across the ranks of `group` (torch.distributed NCCL group) when
    records cross GPUs; meta_group (gloo, CPU) carries the small host tables without a device synchronisation.

    transport "pull" (default): consumers map the producers' buffers (CUDA IPC, dfx_ipc_export/open) and pull the
    token ranges over NVLink with copy engines; the unpack kernel reads the producers' record metadata straight
    from peer memory; two device-side NCCL barriers order the pulls against production and reuse.
    transport "nccl": grouped NCCL send/recv of 16-aligned token ranges + packed metadata (dfx_reshard_pack).
    lazy (pull transport): no consumer batch is built; remote segments stay in the producers' memory as
    RemoteSource runs that the consumer's kernels read over NVLink (dfx_ppo_loss_multi), local segments are views.
    The caller runs ConsumerBatch.release() after its last read (the second device barrier).
    templates / template_key (pull, materialized): the store's cache of exchange templates, keyed by the producer
    sizes and every rank's producer-batch signature; on a hit the table all-gather, the per-segment bookkeeping
    and the consumer's host metadata are reused -- one batched copy call, one unpack, two barriers."""
    L = _declare()
    rank = plan.rank
    for p in plan.local_src:
        if p not in sources:
            raise errors.NotReadyError(f"producer group {p} has not been put on rank {rank}")
    any_b = next(iter(sources.values()))[0] if sources else None
    dev = any_b.device if any_b is not None else torch.device("cuda", torch.cuda.current_device())
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    if schema is None:
        if any_b is None:
            raise errors.Error("exchange on a rank without producer groups needs an explicit schema")
        schema = ({k: v.dtype for k, v in any_b.streams.items()}, [c for c in CHANNELS if c in any_b.channels])
    stream_specs, ch_names = schema
    t_ = _mark("", None)
    loc = _src_slices(plan, sources)
    distributed = plan.cross and _distributed(group)
    pull = distributed and transport == "pull"
    tmpl = templates.get(template_key) if (templates is not None and pull and not lazy) else None
    if tmpl is not None:
        tmpl["hits"] = tmpl.get("hits", 0) + 1
        return _exchange_from_template(tmpl, L, dev, st, group, plan)

    # 1. per-segment table filled by the owner: rollouts, tokens, first token mod 16 (NCCL alignment),
    #    and (pull) the absolute token / rollout / record offsets in the owner's arrays
    nseg = len(plan.segs)
    sizes = np.zeros((nseg, 6), np.int64)
    for i, (b, r0, r1, s0, s1, t0, t1) in loc.items():
        sizes[i] = (s1 - s0, t1 - t0, t0 & 15, t0, s0, r0)
    peer_addr, opened = {}, []
    if pull:
        sizes, peer_addr, opened = _gather_pull_tables(plan, loc, sizes, group, meta_group, ch_names, stream_specs)
    elif distributed:
        sizes = all_reduce_host(sizes, group, meta_group, dev)
    t_ = _mark("sizes", t_)

    # 2. consumer layout on this rank: its consumer groups in dp order
    groups = plan.local_dst
    seg_of = {d: [i for i, sg in enumerate(plan.segs) if sg[0] == d] for d in groups}
    rec_off, roll_off, tok_off = [0], [0], [0]
    dst = {}
    for d in groups:
        s_pos, t_pos = roll_off[-1], tok_off[-1]
        for i in seg_of[d]:
            dst[i] = (rec_off[-1] + int(plan.segs[i][2]), s_pos, t_pos)
            s_pos += int(sizes[i, 0])
            t_pos += int(sizes[i, 1])
        rec_off.append(rec_off[-1] + int(plan.dest_counts[d]))
        roll_off.append(s_pos)
        tok_off.append(t_pos)
    order = [i for d in groups for i in seg_of[d]]

    # zero-copy: every needed segment is local, from one batch, contiguous and in order
    if order and all(i in loc for i in order):
        b0 = loc[order[0]][0]
        if all(loc[i][0] is b0 for i in order) and all(loc[order[k]][2] == loc[order[k + 1]][1]
                                                       for k in range(len(order) - 1)):
            r_a, r_b = loc[order[0]][1], loc[order[-1]][2]
            view = b0 if (r_a == 0 and r_b == b0.n_records) else b0.view_records(r_a, r_b)
            if pull:  # peers may pull from us: take part in both barriers
                _sync_if(plan, group, dev)
                sent = sum(int(sizes[i, 1]) for i, (d, p, *_r) in enumerate(plan.segs) if i in loc
                           for r in plan.dst_ranks[d] if r != rank)
                if lazy:  # the closing barrier is issued at release(), in step with the lazy consumers'
                    return ConsumerBatch(view, groups, rec_off, roll_off, True, sent, 0,
                                         release=lambda: _sync_if(plan, group, dev))
                _sync_if(plan, group, dev)
                return ConsumerBatch(view, groups, rec_off, roll_off, True, sent, 0)
            _, sent, recv_b, _ = _p2p(plan, loc, sizes, dev, st, group, ch_names, None)
            return ConsumerBatch(view, groups, rec_off, roll_off, True, sent, recv_b)

    if lazy and pull:
        _sync_if(plan, group, dev)  # every producer's stream has passed its production of these batches
        per_group = []
        for d in groups:
            srcs = []
            for i in seg_of[d]:
                if i in loc:
                    b, r0, r1, s0, s1, t0, t1 = loc[i]
                    srcs.append(b.view_records(r0, r1))
                    continue
                n_roll, n_tok, _, t0, s0, r0 = (int(x) for x in sizes[i])
                src = plan.src_rank[plan.segs[i][1]]
                pa = peer_addr[(src, plan.segs[i][1])]
                addr = {"ids": pa["ids"] + 8 * r0, "group_off": pa["group_off"] + 4 * r0, "cu": pa["cu"] + 8 * s0}
                for name in ch_names:
                    addr["c:" + name] = pa["c:" + name] + 8 * s0
                for k in stream_specs:
                    addr["s:" + k] = pa["s:" + k]
                srcs.append(RemoteSource(src, int(plan.segs[i][4]), n_roll, t0, n_tok, addr))
            per_group.append(srcs)
        recv_b = sum(int(sizes[i, 1]) * sum(torch.empty(0, dtype=dt_).element_size() for dt_ in stream_specs.values())
                     for i in order if i not in loc)
        return ConsumerBatch(None, groups, rec_off, roll_off, False, 0, recv_b, per_group,
                             release=lambda: _sync_if(plan, group, dev), ipc_bases=opened)

    # 3. allocate the consumer batch
    R, S, T = rec_off[-1], roll_off[-1], tok_off[-1]
    out = _alloc_batch(R, S, T, ch_names, stream_specs, dev)
    t_ = _mark("alloc", t_)

    metas = []
    # local segments: token copies on this GPU + metadata straight from the source arrays
    for i in order:
        if i not in loc:
            continue
        b, r0, r1, s0, s1, t0, t1 = loc[i]
        dr, ds, dt = dst[i]
        for k, t in out.streams.items():
            if t1 > t0:
                t[dt:dt + (t1 - t0)].copy_(b.streams[k][t0:t1], non_blocking=True)
        metas.append(_meta(b, r0, r1, s0, ch_names, dr, ds, dt))
    t_ = _mark("local copies", t_)
    sent = recv_b = 0
    recvd = []
    if pull:
        _sync_if(plan, group, dev)  # every producer's stream has passed its production of these batches
        for i in order:
            if i in loc:
                continue
            n_roll, n_tok, _, t0, s0, r0 = (int(x) for x in sizes[i])
            dr, ds, dt = dst[i]
            src = plan.src_rank[plan.segs[i][1]]
            addr = peer_addr[(src, plan.segs[i][1])]
            for k, t in out.streams.items():
                esz = t.element_size()
                _abi.check(L.dfx_copy_async(t.data_ptr() + dt * esz, addr["s:" + k] + t0 * esz, n_tok * esz,
                                            st.cuda_stream))
                recv_b += n_tok * esz
            m = SegMeta()
            m.ids = addr["ids"] + 8 * r0
            m.group_off = addr["group_off"] + 4 * r0
            m.cu = addr["cu"] + 8 * s0
            for c, name in enumerate(ch_names):
                m.ch[c] = addr["c:" + name] + 8 * s0
            m.n_rec, m.n_roll, m.dst_rec, m.dst_roll, m.dst_tok = int(plan.segs[i][4]), n_roll, dr, ds, dt
            metas.append(m)
        sent = sum(int(sizes[i, 1]) * sum(torch.empty(0, dtype=dt_).element_size() for dt_ in stream_specs.values())
                   for i, (d, p, *_r) in enumerate(plan.segs) if i in loc for r in plan.dst_ranks[d] if r != rank)
    else:
        # remote segments: one grouped NCCL P2P call (sends of our segments to peers, receives of theirs)
        recvd, sent, recv_b, staged = _p2p(plan, loc, sizes, dev, st, group, ch_names, (out, dst))
        # place the received 16-aligned supersets at their exact (unaligned) destination offsets
        for i, k, buf in staged:
            head, n_tok = int(sizes[i, 2]), int(sizes[i, 1])
            dt = dst[i][2]
            out.streams[k][dt:dt + n_tok].copy_(buf[head:head + n_tok], non_blocking=True)
        for i, buf in recvd:
            n_rec, n_roll = int(plan.segs[i][4]), int(sizes[i, 0])
            dr, ds, dt = dst[i]
            base = buf.data_ptr()
            m = SegMeta()
            m.ids = base
            m.cu = base + 8 * n_rec
            for c in range(len(ch_names)):
                m.ch[c] = base + 8 * n_rec + 8 * (n_roll + 1) + 8 * c * n_roll
            m.group_off = base + 8 * n_rec + 8 * (n_roll + 1) + 8 * len(ch_names) * n_roll
            m.n_rec, m.n_roll, m.dst_rec, m.dst_roll, m.dst_tok = n_rec, n_roll, dr, ds, dt
            metas.append(m)
    t_ = _mark("transfer", t_)
    if metas:
        segs = (SegMeta * len(metas))(*metas)
        chp = (C.c_void_p * max(1, len(ch_names)))(*[out.channels[c].data_ptr() for c in ch_names])
        _abi.check(L.dfx_reshard_unpack(C.cast(segs, C.c_void_p), len(metas), len(ch_names), out.ids.data_ptr(),
                                        out.group_off.data_ptr(), out.roll_group.data_ptr(), out.cu_seqlens.data_ptr(),
                                        C.cast(chp, C.c_void_p), st.cuda_stream))
        out._keep = [recvd]
    if pull:
        _sync_if(plan, group, dev)  # peers may reuse their buffers once every consumer has pulled
    t_ = _mark("unpack", t_)
    # host offsets of the consumer batch are fetched lazily (PackedBatch.ensure_host_meta): no D2H here
    out.host_group_off, out.host_cu = None, None
    cbatch = ConsumerBatch(out, groups, rec_off, roll_off, False, sent, recv_b, ipc_bases=opened)
    if pull and templates is not None and template_key is not None:
        # record this exchange as a template: every copy as (stream, offset in the consumer stream, source
        # address, bytes), the unpack segments, and (after one D2H, only now) the consumer's host offsets
        copies = []
        for i in order:
            if i in loc:
                b, r0, r1, s0, s1, t0, t1 = loc[i]
                for k, t in out.streams.items():
                    esz = t.element_size()
                    copies.append((k, dst[i][2] * esz, b.streams[k].data_ptr() + t0 * esz, (t1 - t0) * esz))
            else:
                n_roll, n_tok, _, t0, s0, r0 = (int(x) for x in sizes[i])
                addr = peer_addr[(plan.src_rank[plan.segs[i][1]], plan.segs[i][1])]
                for k, t in out.streams.items():
                    esz = t.element_size()
                    copies.append((k, dst[i][2] * esz, addr["s:" + k] + t0 * esz, n_tok * esz))
        out.ensure_host_meta()
        templates[template_key] = {"R": R, "S": S, "T": T, "ch": list(ch_names), "specs": dict(stream_specs),
                                   "copies": copies, "metas": (SegMeta * len(metas))(*metas), "n_metas": len(metas),
                                   "groups": groups, "rec_off": rec_off, "roll_off": roll_off, "sent": sent,
                                   "recv": recv_b, "h_go": out.host_group_off, "h_cu": out.host_cu,
                                   "ipc": cbatch}
        cbatch.template_owned = True  # the template's replays read these mappings: it owns them now
        if len(templates) > 8:
            old_t = templates.pop(next(iter(templates)))
            old_t["ipc"].close_mappings()
    return cbatch


def _exchange_from_template(tm: dict, L, dev, st, group, plan) -> ConsumerBatch:
    """A materialized pull whose producers are exactly those of the template (same memory, extents and
    placement on every rank): fresh consumer buffers, the recorded copies in one call, one unpack."""
    out = _alloc_batch(tm["R"], tm["S"], tm["T"], tm["ch"], tm["specs"], dev)
    base = {k: t.data_ptr() for k, t in out.streams.items()}
    cp = tm["copies"]
    dsts = np.array([base[k] + off for k, off, _, _ in cp], np.uint64)
    srcs = np.array([a for _, _, a, _ in cp], np.uint64)
    nbs = np.array([n for _, _, _, n in cp], np.uint64)
    _sync_if(plan, group, dev)  # every producer's stream has passed its production of these batches
    _abi.check(L.dfx_copy_many(len(cp), dsts.ctypes.data, srcs.ctypes.data, nbs.ctypes.data, st.cuda_stream))
    if tm["n_metas"]:
        chp = (C.c_void_p * max(1, len(tm["ch"])))(*[out.channels[c].data_ptr() for c in tm["ch"]])
        _abi.check(L.dfx_reshard_unpack(C.cast(tm["metas"], C.c_void_p), tm["n_metas"], len(tm["ch"]),
                                        out.ids.data_ptr(), out.group_off.data_ptr(), out.roll_group.data_ptr(),
                                        out.cu_seqlens.data_ptr(), C.cast(chp, C.c_void_p), st.cuda_stream))
    _sync_if(plan, group, dev)  # peers may reuse their buffers once every consumer has pulled
    out.host_group_off, out.host_cu = tm["h_go"], tm["h_cu"]
    return ConsumerBatch(out, tm["groups"], tm["rec_off"], tm["roll_off"], False, tm["sent"], tm["recv"])


def reuse_lazy(prev: ConsumerBatch, group, plan) -> ConsumerBatch:
    """A lazy consumer batch for a step whose producer batches are the ones `prev` mapped (same memory and
    extents on every rank, checked by the store): same sources, fresh ordering barriers."""
    dev = torch.device("cuda", torch.cuda.current_device())
    _sync_if(plan, group, dev)  # every producer's stream has passed its production of these batches
    return ConsumerBatch(None, prev.groups, prev.rec_off, prev.roll_off, False, prev.bytes_sent, prev.bytes_recv,
                         prev.sources, release=lambda: _sync_if(plan, group, dev))


def reuse_zero_copy(prev: ConsumerBatch, plan: Plan, sources: dict, group) -> ConsumerBatch:
    """A lazy step on a rank whose consumer groups were a zero-copy view last time, with every rank's producer
    batches unchanged (the store's template hit, taken by all ranks alike): the same view over this step's
    producer batch (host-only), and the same two barriers as the lazy consumers -- the first now, the second at
    release()."""
    loc = _src_slices(plan, sources)
    order = [i for d in prev.groups for i, sg in enumerate(plan.segs) if sg[0] == d]
    b0, r_a, r_b = loc[order[0]][0], loc[order[0]][1], loc[order[-1]][2]
    view = b0 if (r_a == 0 and r_b == b0.n_records) else b0.view_records(r_a, r_b)
    if not _distributed(group):
        return ConsumerBatch(view, prev.groups, prev.rec_off, prev.roll_off, True, 0, 0)
    dev = view.device
    _sync_if(plan, group, dev)
    return ConsumerBatch(view, prev.groups, prev.rec_off, prev.roll_off, True, prev.bytes_sent, 0,
                         release=lambda: _sync_if(plan, group, dev))


_BARRIER = {}


def _sync_if(plan, group, dev):
    """The exchange's ordering barrier, needed only when some record crosses GPUs: with every consumer group on the
    GPU of its producer groups (box placements on <= 4 GPUs) no rank reads another's memory, stream order alone
    orders production before consumption, and every rank skips it alike (plan.cross is global)."""
    if plan.cross:
        _device_barrier(group, dev)


def _device_barrier(group, dev):
    """Device-side barrier: a 1-element NCCL all-reduce on the current stream (no host synchronisation). When it
    completes on this GPU, every rank's stream has executed everything enqueued before its own barrier."""
    t = _BARRIER.get(dev)
    if t is None:
        t = _BARRIER[dev] = torch.zeros(1, dtype=torch.int32, device=dev)
    torch.distributed.all_reduce(t, group=group)


def _alloc_batch(R, S, T, ch_names, stream_specs, dev) -> PackedBatch:
    """A consumer batch carved out of ONE device allocation (16-byte aligned arrays): one allocator call instead
    of one per array. The stream padding past T is left as is: kernels discard out-of-range lanes."""
    specs = [("ids", torch.int64, R), ("go", torch.int32, R + 1), ("rg", torch.int32, S), ("cu", torch.int64, S + 1)]
    specs += [("c:" + c, torch.float64, S) for c in ch_names]
    specs += [("s:" + k, dt, padded_len(T)) for k, dt in stream_specs.items()]
    offs, off = {}, 0
    for name, dt, n in specs:
        off = (off + 15) & ~15
        offs[name] = off
        off += n * torch.empty(0, dtype=dt).element_size()
    buf = torch.empty(off + 16, dtype=torch.uint8, device=dev)
    arr = {name: buf[offs[name]:offs[name] + n * torch.empty(0, dtype=dt).element_size()].view(dt)
           for name, dt, n in specs}
    return PackedBatch(R, S, 0, T, arr["ids"], arr["go"], arr["rg"], arr["cu"],
                       {c: arr["c:" + c] for c in ch_names}, {k: arr["s:" + k] for k in stream_specs})


def _export(t: torch.Tensor):
    h = (C.c_char * 64)()
    off = C.c_uint64()
    _abi.check(_declare().dfx_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
    return bytes(h), int(off.value)


def _gather_pull_tables(plan: Plan, loc: dict, sizes, group, meta_group, ch_names, stream_specs):
    """One fixed-size int64 all-gather (CPU group) carrying every rank's segment rows and the IPC exports
    (64-byte handle + offset) of its producer batches' arrays; returns the global table and
    {(src rank, producer group): {array: mapped device address}}."""
    L = _declare()
    names = ["ids", "group_off", "cu"] + ["c:" + c for c in ch_names] + ["s:" + k for k in stream_specs]
    nseg, dp_p, na = len(plan.segs), plan.produced.dp, len(names)
    width = nseg * 6 + dp_p * na * 9
    mine = np.zeros(width, np.int64)
    exp = mine[nseg * 6:].reshape(dp_p, na, 9)
    roots = {}
    for i, (b, *_r) in loc.items():
        mine[i * 6:(i + 1) * 6] = sizes[i]
        p = plan.segs[i][1]
        key = id(b)
        if key not in roots:
            arr = {"ids": b.ids, "group_off": b.group_off, "cu": b.cu_seqlens}
            for name in ch_names:
                arr["c:" + name] = b.channels[name]
            for k in stream_specs:
                arr["s:" + k] = b.streams[k]
            rows = np.zeros((na, 9), np.int64)
            for j, n in enumerate(names):
                h, off = _export(arr[n])
                rows[j, :8] = np.frombuffer(h, np.int64)
                rows[j, 8] = off
            roots[key] = rows
        exp[p] = roots[key]
    world = torch.distributed.get_world_size(group)
    cpu = meta_group is not None
    t = torch.from_numpy(mine)
    if not cpu:
        t = t.cuda()
    gathered = [torch.empty_like(t) for _ in range(world)]
    torch.distributed.all_gather(gathered, t, group=meta_group if cpu else group)
    allrows = np.stack([g.cpu().numpy() for g in gathered])
    table = np.zeros_like(sizes)
    for i, (d, p, *_x) in enumerate(plan.segs):
        table[i] = allrows[plan.src_rank[p], i * 6:(i + 1) * 6]
    addr, opened = {}, []
    for i, (d, p, *_x) in enumerate(plan.segs):
        src = plan.src_rank[p]
        if src == plan.rank or plan.rank not in plan.dst_ranks[d] or (src, int(p)) in addr:
            continue
        rows = allrows[src, nseg * 6:].reshape(dp_p, na, 9)[p]
        out = {}
        for j, n in enumerate(names):
            base = C.c_void_p()
            _abi.check(L.dfx_ipc_open(rows[j, :8].tobytes(), 64, C.byref(base)))
            opened.append(base.value)
            out[n] = base.value + int(rows[j, 8])
        addr[(src, int(p))] = out
    return table, addr, opened


def all_reduce_host(a: np.ndarray, group, meta_group, dev) -> np.ndarray:
    """Sum a small int64 host table over ranks: over the CPU group when given, else through the device group."""
    t = torch.from_numpy(np.ascontiguousarray(a, np.int64).reshape(-1).copy())
    if meta_group is not None:
        torch.distributed.all_reduce(t, group=meta_group)
        return t.numpy().reshape(a.shape)
    if torch.distributed.get_backend(group) == "nccl":
        t = t.to(dev)
    torch.distributed.all_reduce(t, group=group)
    return t.cpu().numpy().reshape(a.shape)


def _distributed(group) -> bool:
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return False
    return torch.distributed.get_world_size(group) > 1


def _to_device(cstruct, dev) -> torch.Tensor:
    """Small host table (ctypes array) -> device bytes (synchronous H2D: the table is freed right after)."""
    return torch.frombuffer(bytearray(bytes(cstruct)), dtype=torch.uint8).to(dev)


def _meta(b: PackedBatch, r0, r1, s0, ch_names, dr, ds, dt) -> SegMeta:
    m = SegMeta()
    m.ids = b.ids.data_ptr() + 8 * r0
    m.group_off = b.group_off.data_ptr() + 4 * r0
    m.cu = b.cu_seqlens.data_ptr() + 8 * s0
    for c, name in enumerate(ch_names):
        m.ch[c] = b.channels[name].data_ptr() + 8 * s0
    m.n_rec, m.n_roll = r1 - r0, int(b.host_group_off[r1]) - s0
    m.dst_rec, m.dst_roll, m.dst_tok = dr, ds, dt
    return m


def _p2p(plan: Plan, loc: dict, sizes, dev, st, group, ch_names, recv_into):
    """Post every cross-GPU send of locally held segments and (when recv_into=(consumer batch, dst offsets) is
    given) every receive of remote segments this rank needs, as ONE grouped NCCL call. Per (src, dst) pair the
    messages are posted in segment order on both sides: packed metadata, then token streams sorted by name.
    Token streams travel as 16-token-aligned supersets [t0 & ~15, align16(t1)) straight from the producer's
    streams into aligned staging buffers (NCCL P2P runs ~2.5x slower on misaligned buffers, measured on B200);
    the caller places the exact range. Returns ([(segment, packed metadata buffer)], bytes sent, bytes received,
    [(segment, stream name, staging buffer)])."""
    if not plan.cross or not _distributed(group):
        return [], 0, 0, []
    t_ = _mark("", None)
    L = _declare()
    ops, recvd, to_pack, staged = [], [], [], []
    sent = recv_b = 0
    me = plan.rank
    for i, (d, p, dr, sr, n) in enumerate(plan.segs):
        src = plan.src_rank[p]
        for r in plan.dst_ranks[d]:
            if src == me and r != me:
                b, r0, r1, s0, s1, t0, t1 = loc[i]
                nb = L.dfx_reshard_pack_bytes(r1 - r0, s1 - s0, len(ch_names))
                buf = torch.empty(nb, dtype=torch.uint8, device=dev)
                to_pack.append((_meta(b, r0, r1, s0, ch_names, 0, 0, 0), buf))
                ops.append(torch.distributed.P2POp(torch.distributed.isend, buf, r, group))
                sent += nb
                if t1 > t0:
                    t0a, t1a = t0 & ~15, (t1 + 15) & ~15
                    for k in sorted(b.streams):
                        sl = b.streams[k][t0a:t1a]
                        ops.append(torch.distributed.P2POp(torch.distributed.isend, sl, r, group))
                        sent += sl.numel() * sl.element_size()
            elif r == me and src != me and recv_into is not None:
                out, dst = recv_into
                dr_, ds, dt = dst[i]
                n_tok = int(sizes[i, 1])
                nb = L.dfx_reshard_pack_bytes(int(n), int(sizes[i, 0]), len(ch_names))
                buf = torch.empty(nb, dtype=torch.uint8, device=dev)
                recvd.append((i, buf))
                ops.append(torch.distributed.P2POp(torch.distributed.irecv, buf, src, group))
                recv_b += nb
                if n_tok:
                    head = int(sizes[i, 2])
                    n_al = ((head + n_tok + 15) & ~15)
                    for k in sorted(out.streams):
                        buf_k = torch.empty(n_al, dtype=out.streams[k].dtype, device=dev)
                        staged.append((i, k, buf_k))
                        ops.append(torch.distributed.P2POp(torch.distributed.irecv, buf_k, src, group))
                        recv_b += buf_k.numel() * buf_k.element_size()
    t_ = _mark("p2p:post-prep", t_)
    if to_pack:
        segs = (SegMeta * len(to_pack))(*[m for m, _ in to_pack])
        outp = (C.c_void_p * len(to_pack))(*[b.data_ptr() for _, b in to_pack])
        _abi.check(L.dfx_reshard_pack(C.cast(segs, C.c_void_p), len(to_pack), len(ch_names), C.cast(outp, C.c_void_p),
                                      st.cuda_stream))
    t_ = _mark("p2p:pack", t_)
    if ops:
        for w in torch.distributed.batch_isend_irecv(ops):
            w.wait()
    t_ = _mark("p2p:nccl (%d ops)" % len(ops), t_)
    return recvd, sent, recv_b, staged
