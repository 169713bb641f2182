"""DP m->n reshard of device-resident packed batches (distflow/data_plane.hpp BufferStore exchange/get).

BoxReshard: the bench's placement -- one DataBuffer per box (B = 1, W = 8 logical workers), worker w on GPU
w // (8 / P). Producer layout dp_p with tp 1, consumer layout dp_c with tp = 8 / dp_c.
Destination group d receives (L_0 || ... || L_7)[d*G/dp_c, (d+1)*G/dp_c) (SURVEY.md App. A, B = 1), i.e. the
producer groups [d*8/dp_c, (d+1)*8/dp_c). When every TP worker of d sits on the GPU that already holds those
producer groups (P <= 8/tp_c... here P <= 4) the consumer batch is a zero-copy view of the producer batch.
"""
from __future__ import annotations

import numpy as np
import torch

from . import errors


class BoxReshard:
    def __init__(self, world: int, rank: int, device, producer_dp: int = 8, consumer_dp: int = 4, workers: int = 8):
        if workers % world:
            raise errors.LayoutError(f"{workers} logical workers cannot be spread over {world} GPUs")
        if workers % producer_dp or workers % consumer_dp:
            raise errors.LayoutError("dp must divide the logical world")
        self.world, self.rank, self.device = world, rank, torch.device(device)
        self.W, self.dp_p, self.dp_c = workers, producer_dp, consumer_dp
        self.tp_c = workers // consumer_dp
        self.wpg = workers // world  # logical workers per GPU
        self.local = self.tp_c <= self.wpg  # every consumer group's TP workers share this GPU
        self._lgo_cache = {}
        self.launches_per_step = 0 if self.local else 4

    def describe(self) -> str:
        mode = ("zero-copy views (all TP workers of each consumer group and its producer groups share a GPU)"
                if self.local else "TP-partner exchange over NVLink (NCCL P2P) + metadata rebase")
        return (f"B=1 W={self.W}: dp{self.dp_p}(tp1) -> dp{self.dp_c}(tp{self.tp_c}) over {self.world} GPU; {mode}")

    def local_consumer_groups(self):
        """Consumer DP groups with at least one TP worker on this GPU (dp_rank = worker // tp_c)."""
        first_w, last_w = self.rank * self.wpg, (self.rank + 1) * self.wpg
        return sorted({w // self.tp_c for w in range(first_w, last_w)})

    def exchange(self, batch, ctx):
        """Returns (consumer batch on this GPU, rollout offsets of its consumer groups)."""
        if not self.local:
            raise errors.Error("BoxReshard: cross-GPU exchange requires reshard.Reshard (general executor)")
        groups = self.local_consumer_groups()
        key = (id(batch.host_group_off), batch.n_records)
        lgo = self._lgo_cache.get(key)
        if lgo is None:
            # producer groups on this GPU hold equal record counts; consumer group d = producer groups
            # [d*pg, (d+1)*pg) with pg = dp_p/dp_c, all local here, in order
            n_local_prod = self.dp_p // self.world
            per_prod = batch.n_records // n_local_prod
            per_cons = per_prod * (self.dp_p // self.dp_c)
            rec_off = [i * per_cons for i in range(len(groups) + 1)]
            if rec_off[-1] != batch.n_records:
                raise errors.IndivisibleError.of("store holdings", batch.n_records, len(groups))
            lgo = [int(batch.host_group_off[r]) for r in rec_off]
            self._lgo_cache = {key: lgo}
        return batch, lgo
