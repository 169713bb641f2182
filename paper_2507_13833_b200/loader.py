"""Dataset sharding and the per-DP-group loader: the step before the path.

Mirrors distflow/data_plane.hpp:115-209:
  shard_dataset(dataset_size, dp)      data_plane.hpp:124-135 -- dp equal contiguous ranges, IndivisibleError otherwise
  DataLoader(range, dp, dp_rank, ...)  data_plane.hpp:162-201 -- optional one-time keyed Fisher-Yates shuffle
                                       (keyed_hash(seed, "shuffle", dp_rank, i) % i, :168-173)
  DataLoader.next_batch_ids            data_plane.hpp:177-190 -- idx = (iteration * per_group + j) % shard size
  make_group_loader                    data_plane.hpp:204-209
The reference loads SampleRecords whose only identity is sample_id (the synthetic prompt is a pure function of
(seed, sample_id), data_plane.hpp:51-60, and no hot-path function reads it), so the loader here yields the batch's
sample ids and `next_batch` turns them into a device-resident PackedBatch through PackedBatch.synthetic(ids=...)
(rollout lengths/channels by the reference's keyed hashes, token streams by dfx_synth_tokens on the device).
Ids are bit-identical to the reference loader's (tests/test_loader.py, against oracle/_ref).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import synth
from .errors import Error, IndivisibleError


@dataclass(frozen=True)
class ShardRange:
    """distflow::ShardRange (data_plane.hpp:117-122): rows [first, last)."""

    first: int
    last: int

    def size(self) -> int:
        return self.last - self.first


def shard_dataset(dataset_size: int, dp: int) -> list[ShardRange]:
    """data_plane.hpp:124-135."""
    if dp == 0 or dataset_size % dp != 0:
        raise IndivisibleError.of("dataset size", dataset_size, dp)
    per = dataset_size // dp
    return [ShardRange(g * per, (g + 1) * per) for g in range(dp)]


class DataLoader:
    """One DP group's slice of a synthetic dataset (data_plane.hpp:162-201). Reads are a pure function of
    (iteration, global batch); the cursor wraps at the shard end."""

    def __init__(self, shard: ShardRange, dp: int, dp_rank: int, seed: int, shuffle: bool = False):
        self.shard, self.dp, self.dp_rank, self.seed = shard, dp, dp_rank, seed
        n = shard.size()
        order = np.arange(n, dtype=np.int64)
        if shuffle and n > 1:
            i = np.arange(n, 1, -1, dtype=np.uint64)  # i = n .. 2, the reference's swap order
            js = (synth.keyed_hash(seed, "shuffle", dp_rank, i) % i).astype(np.int64)
            for i_, j in zip(range(n, 1, -1), js.tolist()):
                order[i_ - 1], order[j] = order[j], order[i_ - 1]
        self.order = order

    def shard_size(self) -> int:
        return self.shard.size()

    def next_batch_ids(self, iteration: int, global_batch: int) -> np.ndarray:
        """Sample ids of next_batch(iteration, global_batch) (data_plane.hpp:177-190), uint64."""
        if global_batch % self.dp != 0:
            raise IndivisibleError.of("global batch", global_batch, self.dp)
        per_group = global_batch // self.dp
        n = self.shard.size()
        if n == 0:
            raise Error("loader shard is empty")
        idx = (np.uint64(iteration) * np.uint64(per_group) + np.arange(per_group, dtype=np.uint64)) % np.uint64(n)
        return (np.uint64(self.shard.first) + self.order[idx.astype(np.int64)].astype(np.uint64)).astype(np.uint64)

    def next_batch(self, iteration: int, global_batch: int, n_roll: int, dist: synth.TokenDist, device="cuda",
                   streams=("lp", "old_lp", "ref_lp", "mask"), stream=None):
        """The batch as a device-resident PackedBatch (generation included; see the module docstring)."""
        from .packed import PackedBatch
        ids = self.next_batch_ids(iteration, global_batch)
        return PackedBatch.synthetic(self.seed, len(ids), n_roll, dist, device=device, ids=ids, streams=streams,
                                     stream=stream)


def make_group_loader(dataset_size: int, dp: int, dp_rank: int, seed: int, shuffle: bool = False) -> DataLoader:
    """data_plane.hpp:204-209 (synthetic dataset of `dataset_size` rows)."""
    ranges = shard_dataset(dataset_size, dp)
    if not 0 <= dp_rank < len(ranges):
        raise IndexError(f"dp_rank {dp_rank} out of range for dp {dp}")
    return DataLoader(ranges[dp_rank], dp, dp_rank, seed, shuffle)
