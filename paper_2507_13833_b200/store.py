"""DeviceBufferStore: the reference BufferStore's contract (distflow/data_plane.hpp:225-457) over device batches.

One instance per process (GPU). The logical workers it serves are the ones the topology maps to this GPU. The
exchange itself is reshard.exchange (SPMD across GPUs). Kept from the reference, with its error types:
  put        TP != 0 puts are suppressed and counted (:245-248); a producer group must be local (:249-254, "not
             local to node" -> here "not local to rank"); a second put for the same group raises (:256-258);
             iterations below the low-water mark raise StaleIterationError (:241-244)
  get        runs ensure_ready, then returns the destination group's slice; TP peers on one GPU share one
             zero-copy view of identical bytes (:266-292); a non-local destination raises
  ensure_ready  once per (stage, iteration), when every local producer group has put; a missing put raises
             NotReadyError naming the outstanding count (:340-344) -- a single-threaded rank cannot wait for it
  worker_done   when every local logical worker reported, entries at or below the iteration are purged and the
             low-water mark advances (:351-367)
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import errors
from .packed import PackedBatch
from .reshard import ConsumerBatch, Layout, Plan, Topology, exchange, reuse_lazy, reuse_zero_copy


def _signature(batches) -> int:
    """A 63-bit digest of what a lazy exchange reads from this rank's producer batches: device addresses of every
    array, extents, and a checksum of the host offsets. Equal digests on every rank => last step's mapping holds."""
    import numpy as np

    h = []
    for b in batches:
        root = b.parent if b.parent is not None else b
        arrs = [root.ids, root.cu_seqlens] + [root.channels[k] for k in sorted(root.channels)] + \
               [root.streams[k] for k in sorted(root.streams)]
        h += [t.data_ptr() for t in arrs] + [b.n_records, b.n_rollouts, b.token_base, b.token_span, b.parent_rec]
        b.ensure_host_meta()
        w = np.arange(len(b.host_cu), dtype=np.int64) % 1021 + 1
        h += [int(np.dot(b.host_cu, w)), int(np.dot(b.host_group_off, w[:len(b.host_group_off)]))]
    return hash(tuple(h)) & 0x7FFFFFFFFFFFFFFF


@dataclass
class StoreStagePlan:
    """distflow::StoreStagePlan (data_plane.hpp:216-220)."""
    produced: Layout
    consumed: Layout | None = None


@dataclass
class _Entry:
    by_group: dict = field(default_factory=dict)   # dp -> PackedBatch
    ready: ConsumerBatch | None = None
    consumed: Layout | None = None


class DeviceBufferStore:
    def __init__(self, topo: Topology, rank: int, stages: dict, group=None, stream=None, meta_group=None,
                 transport: str = "pull", schema=None):
        self.topo, self.rank, self.stages, self.group, self.stream = topo, rank, dict(stages), group, stream
        self.schema = schema  # ({stream: dtype}, [channels]): needed on ranks that hold no producer group
        self.transport = transport  # "pull" (NVLink peer pulls) or "nccl" (grouped send/recv)
        self.meta_group = meta_group  # CPU (gloo) group for host metadata; data moves over `group` (NCCL)
        self.local_workers = [w for w in range(topo.world) if topo.gpu_of_worker[w] == rank]
        self._entries: dict = {}
        self._done: dict = {}
        self._plans: dict = {}       # (stage, consumed layout, counts) -> Plan
        self._templates: dict = {}   # stage -> (key, lazy ConsumerBatch) for reuse when nothing changed
        self._mat_templates: dict = {}  # (plan key, signatures) -> materialized pull template (reshard.exchange)
        self.template_hits = 0
        self._retired: list = []     # replaced lazy templates whose peer mappings close at the next worker_done
        self.low_water = 0
        self.suppressed = 0
        self.bytes_sent = 0
        self.bytes_recv = 0

    def _plan(self, stage: str) -> StoreStagePlan:
        sp = self.stages.get(stage)
        if sp is None:
            raise errors.UnknownStageError(f"stage '{stage}' not in plan")
        return sp

    def _stale(self, what: str, iteration: int):
        if iteration < self.low_water:
            raise errors.StaleIterationError(f"{what} for iteration {iteration} below low water {self.low_water}")

    def put(self, stage: str, iteration: int, dp_rank: int, tp_rank: int, batch: PackedBatch) -> bool:
        sp = self._plan(stage)
        self._stale("put", iteration)
        if tp_rank != 0:
            self.suppressed += 1
            return False
        if self.topo.gpu_of_worker[sp.produced.group_lead(dp_rank)] != self.rank:
            raise errors.Error(f"put from dp group {dp_rank} not local to rank {self.rank}")
        e = self._entries.setdefault((stage, iteration), _Entry())
        if dp_rank in e.by_group:
            raise errors.Error(f"duplicate put for stage '{stage}' group {dp_rank}")
        e.by_group[dp_rank] = batch
        return True

    def ensure_ready(self, stage: str, iteration: int, fallback_to_layout: Layout, lazy: bool = False) -> ConsumerBatch:
        sp = self._plan(stage)
        self._stale("get", iteration)
        to = sp.consumed or fallback_to_layout
        e = self._entries.setdefault((stage, iteration), _Entry())
        if e.ready is not None:
            return e.ready
        local = [p for p in range(sp.produced.dp)
                 if self.topo.gpu_of_worker[sp.produced.group_lead(p)] == self.rank]
        missing = [p for p in local if p not in e.by_group]
        if missing:
            raise errors.NotReadyError(f"stage '{stage}' iteration {iteration} not ready: {len(missing)} puts "
                                       "outstanding")
        counts = [e.by_group[p].n_records if p in e.by_group else 0 for p in range(sp.produced.dp)]
        # every rank must agree on the producer group sizes; ranks only know their own -> the plan needs them.
        # One small host all-gather carries the counts and a signature of every rank's producer batches.
        sig = _signature([e.by_group[p] for p in local]) if (lazy or self.transport == "pull") else 0
        counts, sigs = self._agree_counts(counts, local, sig)
        pkey = (stage, to, tuple(counts))
        plan = self._plans.get(pkey)
        if plan is None:
            plan = self._plans[pkey] = Plan(self.topo, sp.produced, to, counts, self.rank)
        sources = {p: (e.by_group[p], 0) for p in local}
        tkey = (pkey, tuple(sigs))
        tmpl = self._templates.get(stage)
        if lazy and tmpl is not None and tmpl[0] == tkey:
            # same producer batches everywhere as last time (same memory, same extents): reuse the mapped
            # consumer sources, no table exchange -- only the ordering barriers. tkey holds every rank's
            # signature and every rank records a template after every lazy exchange (zero-copy ones too), so
            # all ranks take this branch together and issue the same collectives
            prev = tmpl[1]
            e.ready = (reuse_zero_copy(prev, plan, sources, self.group) if prev.sources is None
                       else reuse_lazy(prev, self.group, plan))
            self.template_hits += 1
        else:
            e.ready = exchange(plan, sources, stream=self.stream, group=self.group, schema=self.schema,
                               meta_group=self.meta_group, transport=self.transport, lazy=lazy,
                               templates=self._mat_templates, template_key=tkey)
            if lazy:
                if tmpl is not None:
                    self._retired.append(tmpl[1])  # its mappings close once this iteration retires
                self._templates[stage] = (tkey, e.ready)
                e.ready.template_owned = True
        e.consumed = to
        e.by_group = {}
        self.bytes_sent += e.ready.bytes_sent
        self.bytes_recv += e.ready.bytes_recv
        return e.ready

    def _agree_counts(self, counts, local, sig=0):
        """Producer group record counts are known only to their owners; every rank needs all of them. Returns
        (counts, per-rank signatures) from one all-gather (CPU group when available)."""
        import numpy as np
        import torch
        import torch.distributed as dist

        from .reshard import _distributed
        if not _distributed(self.group):
            return counts, [sig]
        mine = np.array([c if p in local else 0 for p, c in enumerate(counts)] + [sig], np.int64)
        t = torch.from_numpy(mine)
        g = self.meta_group
        if g is None:
            t = t.to(torch.device("cuda", torch.cuda.current_device()))
            g = self.group
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size(g))]
        dist.all_gather(parts, t, group=g)
        rows = np.stack([x.cpu().numpy() for x in parts])
        return rows[:, :-1].sum(axis=0).tolist(), rows[:, -1].tolist()

    def get(self, stage: str, iteration: int, dest_dp_rank: int, to_layout: Layout) -> PackedBatch:
        ready = self.ensure_ready(stage, iteration, to_layout)
        if ready.batch is None:
            raise errors.Error("get() after a lazy ensure_ready: the consumer batch is mapped, not materialized")
        if dest_dp_rank not in ready.groups:
            raise errors.Error(f"dp group {dest_dp_rank} not local to rank {self.rank}")
        return ready.group_view(dest_dp_rank)

    def worker_done(self, iteration: int) -> None:
        c = self._done.get(iteration, 0) + 1
        if c < len(self.local_workers):
            self._done[iteration] = c
            return
        self._done.pop(iteration, None)
        for k, e in self._entries.items():  # lazy consumers: peers may reuse their buffers after this barrier
            if k[1] <= iteration and e.ready is not None and e.ready.release is not None:
                e.ready.release()
                e.ready.release = None
        self.low_water = max(self.low_water, iteration + 1)
        for k, e in self._entries.items():  # retire the peer mappings of purged, template-less exchanges
            if k[1] < self.low_water and e.ready is not None and not getattr(e.ready, "template_owned", False):
                e.ready.close_mappings()
        for t in self._retired:
            t.close_mappings()
        self._retired = []
        self._entries = {k: v for k, v in self._entries.items() if k[1] >= self.low_water}

    def suppressed_count(self) -> int:
        return self.suppressed
