"""B200-native DistFlow post-rollout hot path: GRPO/GAE advantage, PPO clipped loss + KL, DP m->n reshard.

The compute lives in libdfx.so (sm_100a CUDA, C ABI in include/dfx.h); this package mirrors the reference's
operator API (distflow/functions.hpp StageFn / FunctionRegistry, distflow/data_plane.hpp BufferStore) on top of
it. Importing it loads the library and raises if it is missing -- there is no CPU fallback.
"""
from . import errors  # noqa: F401
from ._abi import lib as _lib

_lib()  # fail loudly at import when the CUDA library is absent

from .functions import (FunctionRegistry, LossConfig, NodeSpec, StageContext, builtin_gpu_registry,  # noqa: E402,F401
                        fn_gae_advantage, fn_group_advantage, gae_ppo_loss, fn_ppo_advantage, fn_train, invoke_node, loss_dict,
                        ppo_loss, ppo_loss_sources, preset_dag, registry_bind, reward_stats, aggregate_metrics,
                        tp_combine_loss)
from .packed import PackedBatch  # noqa: E402,F401
from .loader import DataLoader, ShardRange, make_group_loader, shard_dataset  # noqa: E402,F401
from .synth import TokenDist  # noqa: E402,F401
from . import wire  # noqa: E402,F401

__version__ = "0.1.0"
