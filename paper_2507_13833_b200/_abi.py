"""ctypes bindings for libdfx.so (include/dfx.h). The product path: it fails loudly when the library is missing.

No CPU fallback exists anywhere in this package; without the CUDA library (or without a GPU) every compute call
raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
# DFX_LIB_PATH: an alternative in-tree build of the same library (kernel variant sweeps, tools/build_variant.py)
LIB_PATH = os.environ.get("DFX_LIB_PATH") or os.path.join(PKG, "lib", "libdfx.so")

P = C.c_void_p
i32, i64, u64, f64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t

KL = {"none": 0, "k1": 1, "k2": 2, "k3": 3}
AGG = {"token-mean": 0, "seq-mean-token-mean": 1, "seq-mean-token-sum": 2}
ADV = {"group": 0, "rollout": 1, "token": 2}


class Packed(C.Structure):
    """dfx_packed (include/dfx.h)."""
    _fields_ = [("n_records", i64), ("n_rollouts", i64), ("group_off", P), ("roll_group", P), ("cu_seqlens", P),
                ("reward", P), ("value", P), ("lp", P), ("old_lp", P), ("ref_lp", P), ("value_tok", P),
                ("token_reward", P), ("mask", P)]


class LossCfg(C.Structure):
    _fields_ = [("clip_low", f64), ("clip_high", f64), ("beta", f64), ("adv_eps", f64), ("kl_type", i32),
                ("agg", i32), ("adv_source", i32), ("whiten", i32)]


class LossArgs(C.Structure):
    _fields_ = [("adv_roll", P), ("adv_tok_in", P), ("whiten_sums", P), ("adv_tok_out", P), ("dlogp", P),
                ("n_loss_groups", i32), ("loss_group_off", P), ("out", P), ("flags", P), ("ev_main_begin", P),
                ("ev_main_end", P)]


class LossSrc(C.Structure):
    """dfx_loss_src (include/dfx.h): one token source of dfx_ppo_loss_multi."""
    _fields_ = [("b", Packed), ("token_base", i64), ("token_span", i64), ("adv_roll", P), ("adv_tok_in", P),
                ("adv_tok_out", P), ("dlogp", P)]


LOSS_OUT_FIELDS = ("loss", "pg_loss", "kl", "clipfrac", "approx_kl", "n_tokens", "n_seqs")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.Error(f"libdfx.so not built at {LIB_PATH}: run `python paper_2507_13833_b200/build.py` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def _declare(L):
    L.dfx_last_error.restype = C.c_char_p
    L.dfx_version.restype = C.c_char_p
    L.dfx_grpo_advantage.argtypes = [C.POINTER(Packed), f64, P, P, P]
    L.dfx_broadcast_advantage.argtypes = [C.POINTER(Packed), i64, i64, P, P, P]
    L.dfx_ppo_advantage.argtypes = [C.POINTER(Packed), P, P]
    L.dfx_gae_workspace_bytes.restype = sz
    L.dfx_gae_workspace_bytes.argtypes = [i64, i64]
    L.dfx_gae.argtypes = [C.POINTER(Packed), i64, i64, f64, f64, P, P, P, P, sz, P]
    L.dfx_gae_ppo_loss_workspace_bytes.restype = sz
    L.dfx_gae_ppo_loss_workspace_bytes.argtypes = [i64, i64]
    L.dfx_gae_ppo_loss.argtypes = [C.POINTER(Packed), i64, i64, f64, f64, C.POINTER(LossCfg), P, P, P, P, sz, P]
    L.dfx_ppo_loss_workspace_bytes.restype = sz
    L.dfx_ppo_loss_workspace_bytes.argtypes = [i64, i64, i32]
    L.dfx_ppo_loss.argtypes = [C.POINTER(Packed), i64, i64, C.POINTER(LossCfg), C.POINTER(LossArgs), P, sz, P]
    L.dfx_ppo_loss_multi_workspace_bytes.restype = sz
    L.dfx_ppo_loss_multi_workspace_bytes.argtypes = [C.POINTER(LossSrc), i32, i32]
    L.dfx_ppo_loss_multi.argtypes = [C.POINTER(LossSrc), i32, C.POINTER(LossCfg), C.POINTER(LossArgs), P, sz, P]
    L.dfx_reward_stats.argtypes = [C.POINTER(Packed), P, P]
    L.dfx_loss_combine.argtypes = [P, i32, i32, C.POINTER(LossCfg), P, P]
    L.dfx_check_flags.argtypes = [P, P]
    L.dfx_synth_tokens.argtypes = [u64, P, i64, i32, P, i64, i64, P, P, P, P, P, P, P, P]
    L.dfx_generate_counts.argtypes = [u64, i32, C.c_uint32, C.c_uint32, C.c_uint32, P, i64, i32, P, P]
    L.dfx_generate_payload.argtypes = [u64, P, i64, i32, P, P, P]
    L.dfx_event_create.argtypes = [C.POINTER(P)]
    L.dfx_event_destroy.argtypes = [P]
    L.dfx_event_record.argtypes = [P, P]
    L.dfx_event_elapsed_ms.argtypes = [P, P, C.POINTER(C.c_float)]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or i32
    for name in ("dfx_grpo_advantage", "dfx_broadcast_advantage", "dfx_ppo_advantage", "dfx_gae", "dfx_ppo_loss",
                 "dfx_gae_ppo_loss",
                 "dfx_ppo_loss_multi",
                 "dfx_check_flags", "dfx_synth_tokens", "dfx_generate_counts", "dfx_generate_payload",
                 "dfx_event_create", "dfx_event_destroy", "dfx_event_record",
                 "dfx_event_elapsed_ms"):
        getattr(L, name).restype = i32


# every symbol include/dfx.h declares (checked by tests/test_abi.py against the header and the .so)
EXPORTS = ("dfx_last_error", "dfx_version", "dfx_grpo_advantage", "dfx_broadcast_advantage", "dfx_ppo_advantage",
           "dfx_gae_workspace_bytes", "dfx_gae", "dfx_ppo_loss_workspace_bytes", "dfx_ppo_loss",
           "dfx_ppo_loss_multi_workspace_bytes", "dfx_ppo_loss_multi", "dfx_check_flags",
           "dfx_synth_tokens", "dfx_generate_counts", "dfx_generate_payload", "dfx_serialize_plan",
           "dfx_serialize_records",
           "dfx_blob_index", "dfx_blob_unpack", "dfx_reward_stats", "dfx_loss_combine", "dfx_copy_batch",
           "dfx_copy_sm", "dfx_view_meta", "dfx_copy_many", "dfx_event_create", "dfx_event_destroy",
           "dfx_event_record", "dfx_event_elapsed_ms")


def check(status: int) -> None:
    """Map a dfx_status to the reference's exception types (distflow/errors.hpp)."""
    if status != 0:
        msg = lib().dfx_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)
