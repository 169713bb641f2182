"""GPU stage functions behind the reference's operator API (distflow/functions.hpp).

Same shapes as the reference: a StageFn is ``fn(node: NodeSpec, batch: PackedBatch, ctx: StageContext) -> None``
that mutates ``batch`` in place (adds channels/streams, leaves the rest untouched), dispatched
through a FunctionRegistry under the reference's registry keys (functions.hpp:184-219), so a DAG built by
``preset_dag`` binds to these GPU nodes unchanged. Errors are the reference's types (errors.py).

Every compute step calls libdfx.so (csrc/); nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _abi, errors
from .packed import PackedBatch, _ptr

# ---- DAG vocabulary (distflow/dag.hpp:17-71) -------------------------------------------
ROLES = ("ACTOR", "CRITIC", "REWARD", "REFERENCE", "NONE")
NODE_TYPES = ("MODEL_INFERENCE", "MODEL_TRAIN", "COMPUTE")


@dataclass
class NodeSpec:
    """distflow::NodeSpec (dag.hpp:57-71)."""
    node_id: str
    role: str = "NONE"
    node_type: str = "COMPUTE"
    func_tag: str | None = None
    deps: list = field(default_factory=list)

    def dispatch_key(self) -> str:  # dag.hpp:65-68
        return self.func_tag if self.func_tag else f"{self.role}/{self.node_type}"


def preset_dag(algorithm: str) -> list[NodeSpec]:
    """distflow::preset_dag (dag.hpp:310-357): node ids, roles, types, func tags and deps of the presets."""
    n = NodeSpec
    a = algorithm.lower()
    if a == "ppo":
        return [n("actor_generate", "ACTOR", "MODEL_INFERENCE", "actor_generate"),
                n("ref_inference", "REFERENCE", "MODEL_INFERENCE", "ref_logprob", ["actor_generate"]),
                n("critic_inference", "CRITIC", "MODEL_INFERENCE", "value_inference", ["actor_generate"]),
                n("reward_compute", "REWARD", "COMPUTE", "reward_compute", ["actor_generate"]),
                n("advantage_compute", "NONE", "COMPUTE", "ppo_advantage",
                  ["ref_inference", "critic_inference", "reward_compute"]),
                n("actor_train", "ACTOR", "MODEL_TRAIN", "train_actor", ["advantage_compute"]),
                n("critic_train", "CRITIC", "MODEL_TRAIN", "train_critic", ["advantage_compute"])]
    if a == "grpo":
        return [n("actor_generate", "ACTOR", "MODEL_INFERENCE", "actor_generate"),
                n("ref_inference", "REFERENCE", "MODEL_INFERENCE", "ref_logprob", ["actor_generate"]),
                n("reward_compute", "REWARD", "COMPUTE", "reward_compute", ["actor_generate"]),
                n("group_advantage_compute", "NONE", "COMPUTE", "group_advantage", ["ref_inference", "reward_compute"]),
                n("actor_train", "ACTOR", "MODEL_TRAIN", "train_actor", ["group_advantage_compute"])]
    raise errors.Error(f"unknown algorithm '{algorithm}'")


# ---- context -------------------------------------------------------------------------------
@dataclass
class LossConfig:
    clip_low: float = 0.2
    clip_high: float = 0.2
    beta: float = 0.001
    kl: str = "k3"
    agg: str = "token-mean"
    whiten: bool = False
    want_grad: bool = False


class Workspace:
    """Caching device scratch, zero-filled at allocation (libdfx kernels leave their tickets zeroed)."""

    def __init__(self):
        self._bufs: dict = {}

    def const(self, key, make):
        """Small device constants (e.g. loss-group offsets) built once and reused."""
        t = self._bufs.get(key)
        if t is None:
            t = make()
            self._bufs[key] = t
        return t

    def get(self, key: str, nbytes: int, device) -> torch.Tensor:
        t = self._bufs.get(key)
        if t is None or t.numel() < nbytes or t.device != torch.device(device):
            t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
            self._bufs[key] = t
        return t


@dataclass
class StageContext:
    """distflow::StageContext (functions.hpp:55-61) + the GPU path's loss/GAE settings and stream."""
    run_seed: int = 0
    advantage_eps: float = 1e-6
    model_versions: dict | None = None
    loss: LossConfig = field(default_factory=LossConfig)
    gae_gamma: float = 1.0
    gae_lambda: float = 0.95
    stream: torch.cuda.Stream | None = None
    workspace: Workspace = field(default_factory=Workspace)

    def cuda_stream(self, device) -> int:
        s = self.stream if self.stream is not None else torch.cuda.current_stream(device)
        return s.cuda_stream


StageFn = Callable[[NodeSpec, PackedBatch, StageContext], None]


def _on_batch_device(pos: int):
    """libdfx launches on the calling thread's current device; run the wrapped op with the batch's device current
    (like torch's DeviceGuard) so one process can drive batches on several GPUs."""
    def deco(fn):
        import functools

        @functools.wraps(fn)
        def run(*args, **kwargs):
            dev = args[pos].device
            if dev.type != "cuda" or dev.index == torch.cuda.current_device():
                return fn(*args, **kwargs)
            with torch.cuda.device(dev):
                return fn(*args, **kwargs)
        return run
    return deco


# ---- checks mirroring detail::require_rollouts / channel_of (functions.hpp:82-93) ---------------
def _require_rollouts(batch: PackedBatch) -> None:
    go = batch.host_group_off
    if go is not None and batch.n_records and (np.diff(go) <= 0).any():
        r = int(np.argmax(np.diff(go) <= 0))
        sid = int(batch.ids[r].item()) & 0xFFFFFFFFFFFFFFFF
        raise errors.MissingRolloutsError(f"record {sid} has no rollouts; generation has not run")


def _channel(batch: PackedBatch, name: str) -> torch.Tensor:
    t = batch.channels.get(name)
    if t is None:
        raise errors.MissingChannelError(name)
    return t


def _stream(batch: PackedBatch, name: str) -> torch.Tensor:
    t = batch.streams.get(name)
    if t is None:
        raise errors.MissingChannelError(name)
    return t


def _reuse_channel(batch: PackedBatch, name: str) -> torch.Tensor:
    """The f64 rollout channel to (over)write: the batch's existing one when it is its own storage of the right
    shape (a stable address for peers that map it), else a fresh tensor. The reference overwrites the channel the
    same way (functions.hpp:159, :170)."""
    t = batch.channels.get(name)
    if t is not None and t.dtype == torch.float64 and t.numel() == batch.n_rollouts and t.is_contiguous() \
            and t.device == batch.device and (batch.parent is None or name not in batch.parent.channels):
        return t
    return torch.empty(batch.n_rollouts, dtype=torch.float64, device=batch.device)


# ---- stage functions ------------------------------------------------------------------------
@_on_batch_device(1)
def fn_group_advantage(node: NodeSpec, batch: PackedBatch, ctx: StageContext) -> None:
    """GPU fn_group_advantage (functions.hpp:143-161): f64, bit-identical; writes channel 'advantage'."""
    _require_rollouts(batch)
    _channel(batch, "reward")
    adv = _reuse_channel(batch, "advantage")
    st = batch.struct()
    _abi.check(_abi.lib().dfx_grpo_advantage(C.byref(st), float(ctx.advantage_eps), _ptr(adv), None,
                                             ctx.cuda_stream(batch.device)))
    batch.channels["advantage"] = adv


@_on_batch_device(1)
def fn_ppo_advantage(node: NodeSpec, batch: PackedBatch, ctx: StageContext) -> None:
    """GPU fn_ppo_advantage (functions.hpp:163-172): advantage = reward - value."""
    _require_rollouts(batch)
    _channel(batch, "reward")
    _channel(batch, "value")
    adv = _reuse_channel(batch, "advantage")
    st = batch.struct()
    _abi.check(_abi.lib().dfx_ppo_advantage(C.byref(st), _ptr(adv), ctx.cuda_stream(batch.device)))
    batch.channels["advantage"] = adv


@_on_batch_device(0)
def broadcast_advantage(batch: PackedBatch, ctx: StageContext) -> torch.Tensor:
    """Per-token advantage stream adv_tok[t] = mask[t] ? f32(advantage[s]) : 0."""
    adv = _channel(batch, "advantage")
    _stream(batch, "mask")
    out = torch.zeros_like(batch.streams["mask"], dtype=torch.float32)
    st = batch.struct()
    _abi.check(_abi.lib().dfx_broadcast_advantage(C.byref(st), batch.token_base, batch.token_span, _ptr(adv),
                                                  _ptr(out), ctx.cuda_stream(batch.device)))
    batch.streams["advantage"] = out
    return out


@_on_batch_device(1)
def fn_gae_advantage(node: NodeSpec, batch: PackedBatch, ctx: StageContext) -> None:
    """GAE reverse scan (new func tag 'gae_advantage'): token streams 'advantage', 'returns' + whitening sums."""
    _require_rollouts(batch)
    for n in ("token_reward", "value_tok", "mask"):
        _stream(batch, n)
    like = batch.streams["token_reward"]
    adv = torch.empty_like(like)  # every token of the span is written
    ret = torch.empty_like(like)
    wsum = torch.empty(3, dtype=torch.float64, device=batch.device)  # written by the call (memset if empty)
    nbytes = _abi.lib().dfx_gae_workspace_bytes(batch.n_rollouts, batch.token_span)
    ws = ctx.workspace.get("gae", nbytes, batch.device)
    st = batch.struct()
    _abi.check(_abi.lib().dfx_gae(C.byref(st), batch.token_base, batch.token_span, float(ctx.gae_gamma),
                                  float(ctx.gae_lambda), _ptr(adv), _ptr(ret), _ptr(wsum), _ptr(ws), ws.numel(),
                                  ctx.cuda_stream(batch.device)))
    batch.streams["advantage"] = adv
    batch.streams["returns"] = ret
    batch.channels["_whiten_sums"] = wsum


@_on_batch_device(0)
def gae_ppo_loss(batch: PackedBatch, ctx: StageContext, want_adv: bool = False) -> dict:
    """GAE fused with the PPO loss (dfx_gae_ppo_loss): one scan pass produces every token's advantage and its
    clipped surrogate + KL terms; the advantage never goes to HBM (want_adv stores it too). Writes the 'returns'
    stream (for the critic). Token-mean aggregation of unwhitened advantages; the two-pass path (fn_gae_advantage +
    ppo_loss) covers whitening and sequence means. Returns {"out": [1, 7] device f64, ["adv"]}."""
    cfg = ctx.loss
    if cfg.whiten or cfg.agg != "token-mean":
        raise errors.Error("gae_ppo_loss: the fused pass is token-mean over unwhitened advantages")
    _require_rollouts(batch)
    for n in ("token_reward", "value_tok", "mask", "lp", "old_lp", "ref_lp"):
        _stream(batch, n)
    like = batch.streams["token_reward"]
    ret = torch.empty_like(like)
    adv = torch.empty_like(like) if want_adv else None
    out = torch.empty(7, dtype=torch.float64, device=batch.device)
    c = _abi.LossCfg(cfg.clip_low, cfg.clip_high, cfg.beta, float(ctx.advantage_eps), _abi.KL[cfg.kl],
                     _abi.AGG[cfg.agg], _abi.ADV["token"], 0)
    L = _abi.lib()
    nbytes = L.dfx_gae_ppo_loss_workspace_bytes(batch.n_rollouts, batch.token_span)
    ws = ctx.workspace.get("gae_loss", nbytes, batch.device)
    st = batch.struct()
    _abi.check(L.dfx_gae_ppo_loss(C.byref(st), batch.token_base, batch.token_span, float(ctx.gae_gamma),
                                  float(ctx.gae_lambda), C.byref(c), _ptr(ret), _ptr(adv), _ptr(out), _ptr(ws),
                                  ws.numel(), ctx.cuda_stream(batch.device)))
    batch.streams["returns"] = ret
    res = {"out": out.view(1, 7)}
    if adv is not None:
        res["adv"] = adv
    return res


@_on_batch_device(0)
def ppo_loss(batch: PackedBatch, ctx: StageContext, adv_source: str | None = None, loss_group_off=None,
             adv_tok_out: bool = False, events=None) -> dict:
    """Fused advantage + clipped surrogate + KL + masked aggregation. Returns device tensors.

    adv_source: 'group' (GRPO stats fused in-kernel from 'reward'), 'rollout' (channel 'advantage'),
    'token' (stream 'advantage', e.g. GAE). Default: token stream if present, else rollout channel, else group.
    """
    cfg = ctx.loss
    if adv_source is None:
        adv_source = ("token" if "advantage" in batch.streams else
                      "rollout" if "advantage" in batch.channels else "group")
    for n in ("lp", "old_lp", "ref_lp", "mask"):
        _stream(batch, n)
    if adv_source == "group":
        _require_rollouts(batch)
        _channel(batch, "reward")
    ng = 1 if loss_group_off is None else len(loss_group_off) - 1
    dev = batch.device
    out = torch.empty(ng * 7, dtype=torch.float64, device=dev)
    adv_roll = None
    if adv_source == "rollout":
        adv_roll = _channel(batch, "advantage")
    elif adv_source == "group":
        adv_roll = torch.empty(batch.n_rollouts, dtype=torch.float64, device=dev)
    adv_tok_in = _stream(batch, "advantage") if adv_source == "token" else None
    whiten = batch.channels.get("_whiten_sums") if cfg.whiten else None
    if cfg.whiten and whiten is None:
        raise errors.Error("whitening needs GAE whitening sums (run gae_advantage first)")
    # every token in [token_base, token_base + token_span) is written by the kernel: no zero-fill needed
    aout = torch.empty_like(batch.streams["lp"]) if adv_tok_out else None
    dlogp = torch.empty_like(batch.streams["lp"]) if cfg.want_grad else None
    lgo = None
    if loss_group_off is not None:
        key = ("lgo", tuple(int(x) for x in loss_group_off))
        lgo = ctx.workspace.const(key, lambda: torch.as_tensor(np.asarray(loss_group_off, np.int32)).to(dev))
    c = _abi.LossCfg(cfg.clip_low, cfg.clip_high, cfg.beta, float(ctx.advantage_eps), _abi.KL[cfg.kl],
                     _abi.AGG[cfg.agg], _abi.ADV[adv_source], int(cfg.whiten))
    ev = events or (None, None)
    a = _abi.LossArgs(_ptr(adv_roll), _ptr(adv_tok_in), _ptr(whiten), _ptr(aout), _ptr(dlogp), ng, _ptr(lgo),
                      _ptr(out), None, ev[0], ev[1])
    nbytes = _abi.lib().dfx_ppo_loss_workspace_bytes(batch.n_rollouts, batch.token_span, ng)
    ws = ctx.workspace.get("loss", nbytes, dev)
    st = batch.struct()
    _abi.check(_abi.lib().dfx_ppo_loss(C.byref(st), batch.token_base, batch.token_span, C.byref(c), C.byref(a),
                                       _ptr(ws), ws.numel(), ctx.cuda_stream(dev)))
    res = {"out": out.view(ng, 7)}
    if adv_source == "group":
        batch.channels["advantage"] = adv_roll
    if aout is not None:
        res["adv_tok"] = aout
    if dlogp is not None:
        res["dlogp"] = dlogp
    return res


def ppo_loss_sources(sources: list, ctx: StageContext, loss_group_off=None, adv_tok_out: bool = False,
                     events=None, device=None) -> dict:
    """dfx_ppo_loss_multi over several token sources in order (local PackedBatch views and/or RemoteSource runs of a
    partner GPU's producer batch, read over NVLink by the streaming kernel): the consumer side of a reshard fused
    with the loss, no copy of the remote tokens. Advantages: each source's 'advantage' rollout channel.
    Returns {"out": [n_groups, 7], "adv_tok": [per-source f32 tensors] (adv_tok_out)}."""
    cfg = ctx.loss
    if cfg.whiten or cfg.want_grad:
        raise errors.Error("ppo_loss_sources: whitening / dlogp are single-source features")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index != torch.cuda.current_device():  # launch on the consumer device (see _on_batch_device)
        with torch.cuda.device(dev):
            return ppo_loss_sources(sources, ctx, loss_group_off, adv_tok_out, events, dev)
    ng = 1 if loss_group_off is None else len(loss_group_off) - 1
    out = torch.empty(ng * 7, dtype=torch.float64, device=dev)
    arr = (_abi.LossSrc * len(sources))()
    keep, aouts = [], []
    for k, src in enumerate(sources):
        x = arr[k]
        if isinstance(src, PackedBatch):
            for n in ("lp", "old_lp", "ref_lp", "mask"):
                _stream(src, n)
            x.b = src.struct()
            x.token_base, x.token_span = src.token_base, src.token_span
            x.adv_roll = _ptr(_channel(src, "advantage"))
        else:  # RemoteSource
            x.b = src.struct()
            x.token_base, x.token_span = src.token_base, src.token_span
            x.adv_roll = src.addr["c:advantage"]
        if adv_tok_out:  # a local array per source, addressed in the source's token coordinates
            a0 = x.token_base & ~3
            buf = torch.empty(((x.token_span + (x.token_base - a0) + 3) // 4) * 4 + 4, dtype=torch.float32,
                              device=dev)
            x.adv_tok_out = buf.data_ptr() - 4 * a0
            aouts.append(buf)
        keep.append(x.b)
    lgo = None
    if loss_group_off is not None:
        key = ("lgo", tuple(int(v) for v in loss_group_off))
        lgo = ctx.workspace.const(key, lambda: torch.as_tensor(np.asarray(loss_group_off, np.int32)).to(dev))
    c = _abi.LossCfg(cfg.clip_low, cfg.clip_high, cfg.beta, float(ctx.advantage_eps), _abi.KL[cfg.kl],
                     _abi.AGG[cfg.agg], _abi.ADV["rollout"], 0)
    ev = events or (None, None)
    a = _abi.LossArgs(None, None, None, None, None, ng, _ptr(lgo), _ptr(out), None, ev[0], ev[1])
    L = _abi.lib()
    nbytes = L.dfx_ppo_loss_multi_workspace_bytes(arr, len(sources), ng)
    ws = ctx.workspace.get("loss_multi", nbytes, dev)
    _abi.check(L.dfx_ppo_loss_multi(arr, len(sources), C.byref(c), C.byref(a), _ptr(ws), ws.numel(),
                                    ctx.cuda_stream(dev)))
    res = {"out": out.view(ng, 7)}
    if adv_tok_out:
        res["adv_tok"] = aouts
    return res


def tp_combine_loss(out: torch.Tensor, ctx: StageContext, group) -> torch.Tensor:
    """TP-split loss: `out` [n_groups, 7] is this rank's loss over the rollouts of each group it holds (ppo_loss /
    ppo_loss_sources); the ranks of `group` (the TP workers of those consumer groups, one process per GPU)
    all-gather their rows (56 B per group over NCCL) and fold them with dfx_loss_combine, so every TP worker ends
    with the group's loss over all its rollouts while each GPU streamed only the tokens it holds -- instead of
    every TP worker streaming the whole group (the partner's half over NVLink)."""
    import torch.distributed as dist
    cfg = ctx.loss
    if cfg.whiten or cfg.want_grad:
        raise errors.Error("tp_combine_loss: whitening / dlogp need group-wide statistics before the loss pass")
    ng = out.shape[0]
    n = dist.get_world_size(group)
    parts = torch.empty(n * ng * 7, dtype=torch.float64, device=out.device)
    dist.all_gather_into_tensor(parts, out.reshape(-1).contiguous(), group=group)
    res = torch.empty(ng * 7, dtype=torch.float64, device=out.device)
    c = _abi.LossCfg(cfg.clip_low, cfg.clip_high, cfg.beta, float(ctx.advantage_eps), _abi.KL[cfg.kl],
                     _abi.AGG[cfg.agg], _abi.ADV["rollout"], 0)
    with torch.cuda.device(out.device):
        _abi.check(_abi.lib().dfx_loss_combine(_ptr(parts), n, ng, C.byref(c), _ptr(res),
                                               ctx.cuda_stream(out.device)))
    return res.view(ng, 7)


@_on_batch_device(0)
def reward_stats(batch: PackedBatch, ctx: StageContext) -> torch.Tensor:
    """detail::record_reward_stats (worker.hpp:177-190) on the device: f64 {count, sum, sum of squares} of the
    rollouts' 'reward' channel."""
    _channel(batch, "reward")
    out = torch.empty(3, dtype=torch.float64, device=batch.device)
    st = batch.struct()
    _abi.check(_abi.lib().dfx_reward_stats(C.byref(st), _ptr(out), ctx.cuda_stream(batch.device)))
    return out


def aggregate_metrics(stats: torch.Tensor, tokens: int, suppressed: int = 0, group=None) -> dict:
    """aggregate_metrics (worker.hpp:275-325) as one scalar all-reduce: every rank contributes its reward stats,
    generation tokens (TP-0 workers only, as the reference) and suppressed puts; every rank returns the cluster
    reward mean / variance (E[r^2] - mean^2, the reference's entropy proxy) and totals."""
    v = torch.cat([stats.to(torch.float64), torch.tensor([float(tokens), float(suppressed)], dtype=torch.float64,
                                                         device=stats.device)])
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.all_reduce(v, group=group)
    n, s, q, t, sup = v.tolist()
    mean = s / n if n else 0.0
    var = q / n - mean * mean if n else 0.0
    return {"reward_count": int(n), "reward_mean": mean, "reward_variance": var, "global_tokens": int(t),
            "suppressed_total": int(sup)}


def loss_dict(out_row: torch.Tensor) -> dict:
    vals = out_row.detach().cpu().tolist()
    return dict(zip(_abi.LOSS_OUT_FIELDS, vals))


def fn_train(node: NodeSpec, batch: PackedBatch, ctx: StageContext) -> None:
    """GPU train node (fills fn_train's slot, functions.hpp:176-182): computes the PPO/GRPO loss on the device,
    stores it as batch.channels['_loss'] (f64[7]), and bumps the role's model version like the reference."""
    if node.role not in ("ACTOR", "CRITIC"):
        raise errors.Error(f"role {node.role} is frozen and cannot train")
    if node.role == "ACTOR":
        res = ppo_loss(batch, ctx)
        batch.channels["_loss"] = res["out"].reshape(-1)
        if "dlogp" in res:
            batch.streams["dlogp"] = res["dlogp"]
    if ctx.model_versions is not None:
        ctx.model_versions[node.role] = ctx.model_versions.get(node.role, 0) + 1


# ---- registry (functions.hpp:184-249) -------------------------------------------------------------
class FunctionRegistry:
    def __init__(self):
        self._fns: dict[str, StageFn] = {}

    def register_fn(self, key: str, fn: StageFn) -> None:
        if key in self._fns:
            raise errors.Error(f"duplicate registration for key '{key}'")  # functions.hpp:187-189
        self._fns[key] = fn

    def find(self, key: str) -> StageFn | None:
        return self._fns.get(key)

    def keys(self):
        return sorted(self._fns)


def builtin_gpu_registry() -> FunctionRegistry:
    """The GPU path under the reference's builtin_registry keys (functions.hpp:201-219) + 'gae_advantage'."""
    reg = FunctionRegistry()
    reg.register_fn("group_advantage", fn_group_advantage)
    reg.register_fn("ppo_advantage", fn_ppo_advantage)
    reg.register_fn("gae_advantage", fn_gae_advantage)
    reg.register_fn("train_actor", fn_train)
    reg.register_fn("train_critic", fn_train)
    reg.register_fn("ACTOR/MODEL_TRAIN", fn_train)
    reg.register_fn("CRITIC/MODEL_TRAIN", fn_train)
    return reg


def registry_bind(chain: list[NodeSpec], registry: FunctionRegistry, layouts: dict):
    """registry_bind (functions.hpp:234-249): UnboundNodeError / LayoutError like the reference."""
    out = []
    for spec in chain:
        key = spec.dispatch_key()
        fn = registry.find(key)
        if fn is None:
            raise errors.UnboundNodeError(spec.node_id, key)
        if spec.node_id not in layouts:
            raise errors.LayoutError(f"no layout for stage '{spec.node_id}'")
        out.append((spec, key, fn, layouts[spec.node_id]))
    return out


def invoke_node(spec: NodeSpec, fn: StageFn, batch: PackedBatch, ctx: StageContext) -> None:
    """detail::invoke_node (worker.hpp:192-200): FunctionError passes through, everything else is wrapped."""
    try:
        fn(spec, batch, ctx)
    except errors.FunctionError:
        raise
    except Exception as e:  # noqa: BLE001
        raise errors.FunctionError(spec.node_id, str(e)) from e
