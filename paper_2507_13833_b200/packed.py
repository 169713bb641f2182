"""Device-resident packed rollout batch: the SoA replacement for SampleBatch (distflow/record.hpp:17-41).

Layout: records r own rollouts [group_off[r], group_off[r+1]); rollout s owns tokens
[cu_seqlens[s], cu_seqlens[s+1]) where cu_seqlens holds ABSOLUTE indices into the token streams. Token streams
are 16-byte aligned and padded so the kernels' aligned 128-bit over-reads stay in bounds. Rollout channels
(reward, value, advantage) are f64 like the reference's channel map values.

torch is used only for device memory and streams (plumbing); all compute goes through libdfx.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi, synth

TOKEN_STREAMS = {"lp": torch.float32, "old_lp": torch.float32, "ref_lp": torch.float32, "value_tok": torch.float32,
                 "token_reward": torch.float32, "mask": torch.uint8, "token_id": torch.int32}
PAD = 16  # elements of slack past the last token (aligned over-read)


def _ptr(t):
    return None if t is None else t.data_ptr()


def padded_len(n_tokens: int) -> int:
    return ((n_tokens + PAD + 15) // 16) * 16


@dataclass
class PackedBatch:
    n_records: int
    n_rollouts: int
    token_base: int
    token_span: int
    ids: torch.Tensor              # int64 (sample_id bits)
    group_off: torch.Tensor        # int32 [R+1], relative (group_off[0] == 0)
    roll_group: torch.Tensor       # int32 [S]
    cu_seqlens: torch.Tensor       # int64 [S+1], absolute token offsets
    channels: dict = field(default_factory=dict)   # name -> f64 [S]
    streams: dict = field(default_factory=dict)    # name -> token stream (shared by views)
    host_group_off: np.ndarray | None = None
    host_cu: np.ndarray | None = None
    meta_blob: np.ndarray | None = None            # host: per-record pre-serialized meta sections (optional)
    meta_off: np.ndarray | None = None
    parent: "PackedBatch | None" = None            # views: the batch whose records [parent_rec, +n) this is
    parent_rec: int = 0

    @property
    def device(self):
        return self.cu_seqlens.device

    @property
    def n_tokens(self) -> int:
        return self.token_span

    # ---- construction -----------------------------------------------------------------
    @staticmethod
    def from_host(ids, group_off, cu_seqlens, channels=None, streams=None, device="cuda", pin=True,
                  stream=None) -> "PackedBatch":
        """H2D copy of a host packed batch (numpy). Token streams are (re)allocated padded and aligned."""
        ids = np.ascontiguousarray(ids, np.uint64)
        group_off = np.ascontiguousarray(group_off, np.int32)
        cu = np.ascontiguousarray(cu_seqlens, np.int64)
        R, S = len(ids), len(cu) - 1
        if group_off[0] != 0 or group_off[-1] != S or len(group_off) != R + 1:
            raise ValueError("group_off must run 0..n_rollouts over n_records+1 entries")
        base, end = int(cu[0]), int(cu[-1])
        dev = torch.device(device)

        def h2d(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            if pin and dev.type == "cuda":
                t = t.pin_memory()
            return t.to(dev, non_blocking=True)

        roll_group = np.repeat(np.arange(R, dtype=np.int32), np.diff(group_off))
        out = PackedBatch(R, S, base, end - base, h2d(ids.view(np.int64)), h2d(group_off), h2d(roll_group), h2d(cu),
                          host_group_off=group_off, host_cu=cu)
        for name, a in (channels or {}).items():
            out.channels[name] = h2d(np.ascontiguousarray(a, np.float64))
        for name, a in (streams or {}).items():
            dt = TOKEN_STREAMS.get(name)
            a = np.asarray(a)
            n = padded_len(end)
            t = torch.zeros(n, dtype=dt if dt is not None else torch.from_numpy(a[:0]).dtype, device=dev)
            src = torch.from_numpy(np.ascontiguousarray(a[:end]))
            if pin and dev.type == "cuda":
                src = src.pin_memory()
            t[:end].copy_(src, non_blocking=True)
            out.streams[name] = t
        return out

    @staticmethod
    def synthetic(seed: int, n_records: int, n_roll: int, dist: synth.TokenDist, device="cuda", first_id: int = 0,
                  streams=("lp", "old_lp", "ref_lp", "mask"), stream=None, ids=None) -> "PackedBatch":
        """Synthetic batch: lengths/channels on the host (keyed hashes), token streams on the device (bit-exact).
        Sample ids are first_id .. first_id + n_records - 1, or `ids` (e.g. a DataLoader batch, loader.py)."""
        if ids is None:
            ids = np.arange(first_id, first_id + n_records, dtype=np.uint64)
        else:
            ids = np.ascontiguousarray(ids, np.uint64)
            if len(ids) != n_records:
                raise ValueError(f"{len(ids)} ids for {n_records} records")
        lens = synth.rollout_lengths(seed, ids, n_roll, dist)
        cu = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens, out=cu[1:])
        go = (np.arange(n_records + 1) * n_roll).astype(np.int32)
        reward, value = synth.rollout_channels(seed, ids, n_roll)
        b = PackedBatch.from_host(ids, go, cu, {"reward": reward, "value": value}, None, device=device)
        n = padded_len(int(cu[-1]))
        for name in streams:
            b.streams[name] = torch.zeros(n, dtype=TOKEN_STREAMS[name], device=b.device)
        g = lambda k: _ptr(b.streams.get(k))  # noqa: E731
        st = stream if stream is not None else torch.cuda.current_stream(b.device).cuda_stream
        with torch.cuda.device(b.device):  # libdfx launches on the current device
            _abi.check(_abi.lib().dfx_synth_tokens(seed, _ptr(b.ids), n_records, n_roll, _ptr(b.cu_seqlens),
                                                   b.token_base, b.token_span, g("lp"), g("old_lp"), g("ref_lp"),
                                                   g("value_tok"), g("token_reward"), g("mask"), g("token_id"), st))
        return b

    # ---- ABI view ------------------------------------------------------------------------
    def ensure_host_meta(self) -> None:
        """Batches produced on the device (e.g. by a reshard) fetch their host offsets lazily, only when a host
        consumer (views, the reshard planner) needs them."""
        if self.host_group_off is None and self.group_off is not None:
            self.host_group_off = self.group_off.cpu().numpy()
            self.host_cu = self.cu_seqlens.cpu().numpy()

    def _materialize(self) -> None:
        """Views defer their rebased record metadata (group_off / roll_group) until a kernel needs it."""
        if self.group_off is None:
            dev = self.device
            go = self.host_group_off
            self.group_off = torch.from_numpy(go).to(dev, non_blocking=True)
            self.roll_group = torch.from_numpy(np.repeat(np.arange(self.n_records, dtype=np.int32),
                                                         np.diff(go))).to(dev, non_blocking=True)

    def struct(self) -> _abi.Packed:
        self._materialize()
        s = self.streams
        ch = self.channels
        return _abi.Packed(self.n_records, self.n_rollouts, _ptr(self.group_off), _ptr(self.roll_group),
                           _ptr(self.cu_seqlens), _ptr(ch.get("reward")), _ptr(ch.get("value")), _ptr(s.get("lp")),
                           _ptr(s.get("old_lp")), _ptr(s.get("ref_lp")), _ptr(s.get("value_tok")),
                           _ptr(s.get("token_reward")), _ptr(s.get("mask")))

    def view_records(self, r0: int, r1: int) -> "PackedBatch":
        """Zero-copy view of records [r0, r1): token streams and channels shared, record metadata rebased."""
        if r0 == 0 and r1 == self.n_records:
            return self
        self.ensure_host_meta()
        go = self.host_group_off
        s0, s1 = int(go[r0]), int(go[r1])
        cu = self.host_cu[s0:s1 + 1]
        ngo = (go[r0:r1 + 1] - s0).astype(np.int32)
        root, base = (self.parent, self.parent_rec) if self.parent is not None else (self, 0)
        return PackedBatch(r1 - r0, s1 - s0, int(cu[0]), int(cu[-1] - cu[0]), self.ids[r0:r1], None, None,
                           self.cu_seqlens[s0:s1 + 1], {k: t[s0:s1] for k, t in self.channels.items()},
                           dict(self.streams), host_group_off=ngo, host_cu=cu, parent=root, parent_rec=base + r0)

    def to_host(self) -> dict:
        """D2H of everything (tests / serialization)."""
        out = {"ids": self.ids.cpu().numpy().view(np.uint64), "group_off": self.group_off.cpu().numpy(),
               "cu_seqlens": self.cu_seqlens.cpu().numpy()}
        for k, t in self.channels.items():
            out[k] = t.cpu().numpy()
        for k, t in self.streams.items():
            out[k] = t.cpu().numpy()
        return out
