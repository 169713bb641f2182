"""ctypes bindings to the CPU oracle (liboracle.so) and to the compiled reference (_ref/libdistflow_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm, as the checker or the timed CPU baseline -- never by the product package (paper_2507_13833_b200/).
See oracle/dfx_oracle.h for what each function restates and its parity status.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdistflow_ref.so")

KL = {"none": 0, "k1": 1, "k2": 2, "k3": 3}
AGG = {"token-mean": 0, "seq-mean-token-mean": 1, "seq-mean-token-sum": 2}
DIST = {"constant": 0, "uniform": 1, "skewed": 2}
STATUS_NAMES = {0: "ok", 1: "Error", 2: "LayoutError", 3: "IndivisibleError", 4: "MissingRolloutsError",
                5: "MissingChannelError", 6: "StaleIterationError", 7: "NotReadyError", 8: "UnknownStageError"}


def build() -> None:
    """Compile the oracle (and the reference shim where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _lib = C.CDLL(ORACLE_SO)
        _declare_oracle(_lib)
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"compiled reference {REF_SO} missing (build it where /root/reference exists)")
        _ref = C.CDLL(REF_SO)
        _declare_ref(_ref)
    return _ref


P = C.c_void_p
u32, u64, i32, i64, f64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double


class TokenDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", u32), ("min", u32), ("max", u32)]


class LossCfg(C.Structure):
    _fields_ = [("clip_low", f64), ("clip_high", f64), ("beta", f64), ("kl_type", C.c_int32),
                ("agg", C.c_int32), ("whiten", C.c_int32), ("pad", C.c_int32)]


class LossOut(C.Structure):
    _fields_ = [(n, f64) for n in ("loss", "pg_loss", "kl", "clipfrac", "approx_kl", "n_tokens", "n_seqs")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def _declare_oracle(L):
    L.dfo_splitmix64.restype = u64
    L.dfo_splitmix64.argtypes = [u64]
    L.dfo_hash_combine.restype = u64
    L.dfo_hash_combine.argtypes = [u64, u64]
    L.dfo_hash_str.restype = u64
    L.dfo_hash_str.argtypes = [u64, C.c_char_p]
    L.dfo_keyed_hash.restype = u64
    L.dfo_keyed_hash.argtypes = [u64, C.c_char_p, C.c_int, P]
    L.dfo_unit_from_hash.restype = f64
    L.dfo_unit_from_hash.argtypes = [u64]
    L.dfo_symmetric_from_hash.restype = f64
    L.dfo_symmetric_from_hash.argtypes = [u64]
    L.dfo_hash_bytes.argtypes = [u64, P, C.c_size_t]
    L.dfo_draw_tokens.argtypes = [C.POINTER(TokenDist), u64, u64, u32, C.POINTER(u32)]
    L.dfo_synth_lengths.argtypes = [C.POINTER(TokenDist), u64, P, u32, u32, P]
    L.dfo_synth_rollout_scalars.argtypes = [u64, P, u32, u32, P, P]
    L.dfo_synth_rollout_scalars.restype = None
    L.dfo_synth_tokens.argtypes = [u64, P, u32, u32, P, P, P, P, P, P, P, P, C.c_int]
    L.dfo_synth_tokens.restype = None
    L.dfo_grpo_advantage.argtypes = [u32, P, P, f64, P]
    L.dfo_ppo_advantage.argtypes = [u32, P, P, P]
    L.dfo_ppo_advantage.restype = None
    L.dfo_broadcast_advantage.argtypes = [u32, P, P, P, P]
    L.dfo_broadcast_advantage.restype = None
    L.dfo_gae.argtypes = [u32, P, P, P, P, f64, f64, P, P, P]
    L.dfo_gae.restype = None
    L.dfo_ppo_loss.argtypes = [u32, P, P, P, P, P, P, C.POINTER(LossCfg), C.POINTER(LossOut), P]
    L.dfo_ppo_loss_mt.argtypes = [u32, P, P, P, P, P, P, C.POINTER(LossCfg), C.POINTER(LossOut), C.c_int]
    L.dfo_reshard_placement.argtypes = [u32, u32, u32, u32, u32, u32, P, P, P]
    L.dfo_serialize_packed.restype = u64
    L.dfo_serialize_packed.argtypes = [u32, P, P, P, P, P, P, C.c_int, P, P, C.c_int, P, P, P]


def _declare_ref(L):
    L.ref_last_error.restype = C.c_char_p
    L.ref_splitmix64.restype = u64
    L.ref_splitmix64.argtypes = [u64]
    L.ref_keyed_hash2.restype = u64
    L.ref_keyed_hash2.argtypes = [u64, C.c_char_p, u64, u64]
    L.ref_keyed_hash3.restype = u64
    L.ref_keyed_hash3.argtypes = [u64, C.c_char_p, u64, u64, u64]
    L.ref_unit_from_hash.restype = f64
    L.ref_unit_from_hash.argtypes = [u64]
    L.ref_symmetric_from_hash.restype = f64
    L.ref_symmetric_from_hash.argtypes = [u64]
    L.ref_hash_bytes.argtypes = [u64, P, C.c_size_t]
    L.ref_hash_bytes.restype = None
    L.ref_generate.argtypes = [u64, C.c_int, u32, u32, u32, u32, u32, P, u32, P, P]
    L.ref_fill_channels.argtypes = [u64, P, u32, u32, P, P, P]
    L.ref_loader_ids.argtypes = [u64, u32, u32, u64, C.c_int, u32, u64, P]
    L.ref_advantage.argtypes = [C.c_int, u32, P, P, P, f64, P]
    L.ref_serialize_packed.restype = i64
    L.ref_serialize_packed.argtypes = [u32, P, P, P, P, P, P, C.c_int, P, P, C.c_int, P, P, P, i64]
    L.ref_reshard.argtypes = [u32, u32, u32, u32, u32, u32, P, u32, P, P, P, P, P, P, C.c_int, P, P,
                              C.c_int, P, P, P, P, P, i64, P, P]
    L.ref_bench.argtypes = [u32, P, P, P, P, P, C.c_int, P, P, u32, u32, u32, u32, u32, u32, C.c_int,
                            C.c_int, P]


def ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))


def _check(code, msg=""):
    if code != 0:
        raise OracleError(code, msg)


def _ref_check(code):
    if code != 0:
        raise OracleError(code, ref().ref_last_error().decode())


# ---- hash ----------------------------------------------------------------------
def splitmix64(z):
    return lib().dfo_splitmix64(z)


def keyed_hash(seed, domain, *counters):
    arr = np.asarray(counters, dtype=np.uint64)
    return lib().dfo_keyed_hash(seed, domain.encode(), len(counters), ptr(arr) if len(counters) else None)


def unit_from_hash(h):
    return lib().dfo_unit_from_hash(h)


def symmetric_from_hash(h):
    return lib().dfo_symmetric_from_hash(h)


def hash_bytes(key, n):
    out = np.zeros(n, np.uint8)
    lib().dfo_hash_bytes(key, ptr(out), n)
    return out


def token_dist(kind="uniform", value=128, lo=64, hi=192):
    return TokenDist(DIST[kind], value, lo, hi)


def draw_tokens(dist: TokenDist, seed, sample_id, rollout):
    out = u32()
    _check(lib().dfo_draw_tokens(C.byref(dist), seed, sample_id, rollout, C.byref(out)))
    return out.value


# ---- synthetic batch -------------------------------------------------------------
class SynthBatch:
    """Host SoA batch in the packed layout the CUDA path consumes."""

    def __init__(self, seed, n_records, n_roll, dist: TokenDist, first_id=0, ids=None, nthreads=None,
                 streams=("lp", "old_lp", "ref_lp", "mask"), pad=64):
        self.seed, self.n_records, self.n_roll = seed, n_records, n_roll
        self.ids = (np.arange(first_id, first_id + n_records, dtype=np.uint64) if ids is None
                    else np.ascontiguousarray(ids, dtype=np.uint64))
        S = n_records * n_roll
        self.n_rollouts = S
        self.cu_seqlens = np.zeros(S + 1, np.int64)
        _check(lib().dfo_synth_lengths(C.byref(dist), seed, ptr(self.ids), n_records, n_roll, ptr(self.cu_seqlens)))
        self.group_off = (np.arange(n_records + 1, dtype=np.int32) * n_roll).astype(np.int32)
        self.roll_group = np.repeat(np.arange(n_records, dtype=np.int32), n_roll)
        self.tok_count = np.diff(self.cu_seqlens).astype(np.uint32)
        self.reward = np.zeros(S, np.float64)
        self.value = np.zeros(S, np.float64)
        lib().dfo_synth_rollout_scalars(seed, ptr(self.ids), n_records, n_roll, ptr(self.reward), ptr(self.value))
        T = int(self.cu_seqlens[-1])
        self.n_tokens = T
        Tp = T + pad  # padded so aligned vector over-reads stay in bounds
        want = set(streams)
        mk = lambda name, dt: np.zeros(Tp, dt) if name in want else None  # noqa: E731
        self.lp, self.old_lp, self.ref_lp = mk("lp", np.float32), mk("old_lp", np.float32), mk("ref_lp", np.float32)
        self.value_tok, self.token_reward = mk("value_tok", np.float32), mk("token_reward", np.float32)
        self.mask, self.token_id = mk("mask", np.uint8), mk("token_id", np.int32)
        nth = nthreads if nthreads is not None else min(os.cpu_count() or 1, 32)
        lib().dfo_synth_tokens(seed, ptr(self.ids), n_records, n_roll, ptr(self.cu_seqlens), ptr(self.lp),
                               ptr(self.old_lp), ptr(self.ref_lp), ptr(self.value_tok), ptr(self.token_reward),
                               ptr(self.mask), ptr(self.token_id), nth)


# ---- advantages / GAE / loss --------------------------------------------------------
def grpo_advantage(group_off, reward, eps=1e-6):
    group_off = np.ascontiguousarray(group_off, np.int32)
    reward = np.ascontiguousarray(reward, np.float64)
    adv = np.zeros_like(reward)
    _check(lib().dfo_grpo_advantage(len(group_off) - 1, ptr(group_off), ptr(reward), eps, ptr(adv)))
    return adv


def ppo_advantage(reward, value):
    reward = np.ascontiguousarray(reward, np.float64)
    value = np.ascontiguousarray(value, np.float64)
    adv = np.zeros_like(reward)
    lib().dfo_ppo_advantage(len(reward), ptr(reward), ptr(value), ptr(adv))
    return adv


def broadcast_advantage(cu_seqlens, adv, mask):
    out = np.zeros(len(mask), np.float32)
    lib().dfo_broadcast_advantage(len(cu_seqlens) - 1, ptr(cu_seqlens), ptr(adv), ptr(mask), ptr(out))
    return out


def gae(cu_seqlens, token_reward, value, mask, gamma=1.0, lam=0.95):
    T = len(mask)
    adv = np.zeros(T, np.float64)
    ret = np.zeros(T, np.float64)
    ws = np.zeros(3, np.float64)
    lib().dfo_gae(len(cu_seqlens) - 1, ptr(cu_seqlens), ptr(token_reward), ptr(value), ptr(mask), gamma, lam,
                  ptr(adv), ptr(ret), ptr(ws))
    return adv, ret, ws


def loss_cfg(clip_low=0.2, clip_high=0.2, beta=0.001, kl="k3", agg="token-mean", whiten=False):
    return LossCfg(clip_low, clip_high, beta, KL[kl], AGG[agg], int(whiten), 0)


def ppo_loss(cu_seqlens, lp, old_lp, ref_lp, adv, mask, cfg: LossCfg, want_grad=False):
    out = LossOut()
    g = np.zeros(len(mask), np.float64) if want_grad else None
    _check(lib().dfo_ppo_loss(len(cu_seqlens) - 1, ptr(cu_seqlens), ptr(lp), ptr(old_lp), ptr(ref_lp), ptr(adv),
                              ptr(mask), C.byref(cfg), C.byref(out), ptr(g)))
    return out.as_dict(), g


def ppo_loss_mt(cu_seqlens, lp, old_lp, ref_lp, adv, mask, cfg: LossCfg, nthreads):
    """Timing-only parallel form (CPU baseline of bench.py); the checker is ppo_loss."""
    out = LossOut()
    _check(lib().dfo_ppo_loss_mt(len(cu_seqlens) - 1, ptr(cu_seqlens), ptr(lp), ptr(old_lp), ptr(ref_lp), ptr(adv),
                                 ptr(mask), C.byref(cfg), C.byref(out), int(nthreads)))
    return out.as_dict()


# ---- reshard ----------------------------------------------------------------------
def reshard_placement(B, W, dp_p, tp_p, dp_c, tp_c, group_counts):
    gc = np.ascontiguousarray(group_counts, np.uint64)
    G = int(gc.sum())
    dc = np.zeros(dp_c, np.uint64)
    idx = np.zeros(max(G, 1), np.uint64)
    _check(lib().dfo_reshard_placement(B, W, dp_p, tp_p, dp_c, tp_c, ptr(gc), ptr(dc), ptr(idx)))
    return dc, idx[:G]


class _Streams:
    """Token streams + rollout channels of a packed batch, marshalled for the C entry points."""

    def __init__(self, streams, channels):
        self.arrs = [np.ascontiguousarray(s) for s in streams]
        self.esz = np.array([a.dtype.itemsize for a in self.arrs], np.uint32)
        self.sp = (C.c_void_p * max(1, len(self.arrs)))(*[a.ctypes.data for a in self.arrs])
        names = sorted(channels)  # std::map order
        self.ch_arrs = [np.ascontiguousarray(channels[n], np.float64) for n in names]
        self.names = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
        self.vals = (C.c_void_p * max(1, len(names)))(*[a.ctypes.data for a in self.ch_arrs])
        self.n_streams, self.n_ch = len(self.arrs), len(names)


def serialize_packed(ids, group_off, tok_count, cu_seqlens, streams=(), channels=None, meta_off=None,
                     meta_blob=None, use_reference=False):
    """serialize_records (record.hpp:151-156) of a packed batch; use_reference=True runs the reference itself."""
    channels = channels or {}
    st = _Streams(streams, channels)
    ids = np.ascontiguousarray(ids, np.uint64)
    group_off = np.ascontiguousarray(group_off, np.int32)
    tok_count = np.ascontiguousarray(tok_count, np.uint32)
    cu_seqlens = np.ascontiguousarray(cu_seqlens, np.int64)
    args = (len(ids), ptr(ids), ptr(meta_off), ptr(meta_blob), ptr(group_off), ptr(tok_count), ptr(cu_seqlens),
            st.n_streams, C.cast(st.sp, C.c_void_p), ptr(st.esz), st.n_ch, C.cast(st.names, C.c_void_p),
            C.cast(st.vals, C.c_void_p))
    if use_reference:
        n = ref().ref_serialize_packed(*args, None, 0)
        out = np.zeros(n, np.uint8)
        ref().ref_serialize_packed(*args, ptr(out), n)
        return out
    n = lib().dfo_serialize_packed(*args, None)
    out = np.zeros(n, np.uint8)
    lib().dfo_serialize_packed(*args, ptr(out))
    return out


def ref_loader_ids(dataset_n, dp, dp_rank, seed, shuffle, iteration, global_batch):
    """The reference DataLoader (make_group_loader(...).next_batch, distflow/data_plane.hpp:124-209) -> the batch's
    sample ids; raises OracleError on the reference's errors."""
    out = np.zeros(max(1, global_batch // max(dp, 1)), np.uint64)
    _ref_check(ref().ref_loader_ids(dataset_n, dp, dp_rank, seed, int(shuffle), iteration, global_batch, ptr(out)))
    return out


def ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, group_counts, ids, group_off=None, tok_count=None, cu_seqlens=None,
                streams=(), channels=None, want_blobs=False, blob_cap=None):
    """Run the reference BufferStore reshard; returns (dest_counts, dest_ids, blobs | None, stats)."""
    R = ref()
    gc = np.ascontiguousarray(group_counts, np.uint64)
    ids = np.ascontiguousarray(ids, np.uint64)
    n = len(ids)
    if group_off is None:
        group_off = np.zeros(n + 1, np.int32)
        tok_count = np.zeros(0, np.uint32)
        cu_seqlens = np.zeros(1, np.int64)
    st = _Streams(streams, channels or {})
    group_off = np.ascontiguousarray(group_off, np.int32)
    tok_count = np.ascontiguousarray(tok_count, np.uint32)
    cu_seqlens = np.ascontiguousarray(cu_seqlens, np.int64)
    dc = np.zeros(dp_c, np.uint64)
    did = np.zeros(max(n, 1), np.uint64)
    stats = np.zeros(2 * B, np.uint64)
    if want_blobs:
        cap = blob_cap or (1 << 20)
        blob = np.zeros(cap, np.uint8)
        boff = np.zeros(dp_c + 1, np.int64)
    else:
        cap, blob, boff = 0, None, None
    code = R.ref_reshard(B, W, dp_p, tp_p, dp_c, tp_c, ptr(gc), n, ptr(ids), None, None, ptr(group_off),
                         ptr(tok_count), ptr(cu_seqlens), st.n_streams, C.cast(st.sp, C.c_void_p), ptr(st.esz),
                         st.n_ch, C.cast(st.names, C.c_void_p), C.cast(st.vals, C.c_void_p), ptr(dc), ptr(did),
                         ptr(blob), cap, ptr(boff), ptr(stats))
    _ref_check(code)
    blobs = None
    if want_blobs:
        blobs = [blob[boff[d]:boff[d + 1]].copy() for d in range(dp_c)]
    return dc, did[:n], blobs, stats


def ref_bench(sb: SynthBatch, streams, B, W, dp_p, tp_p, dp_c, tp_c, nthreads, reps):
    """Time the reference's fn_group_advantage + BufferStore reshard on host cores: (adv_s, reshard_s) per rep."""
    st = _Streams(streams, {})
    out = np.zeros(2, np.float64)
    code = ref().ref_bench(sb.n_records, ptr(sb.ids), ptr(sb.group_off), ptr(sb.tok_count), ptr(sb.cu_seqlens),
                           ptr(sb.reward), st.n_streams, C.cast(st.sp, C.c_void_p), ptr(st.esz), B, W, dp_p, tp_p,
                           dp_c, tp_c, nthreads, reps, ptr(out))
    _ref_check(code)
    return float(out[0]), float(out[1])
