#!/bin/bash
# NCCL point-to-point rate between 2 GPUs (torch NCCL, 67 MB each way) under channel settings (env knobs).
for cfg in "" "NCCL_MIN_P2P_NCHANNELS=16" "NCCL_MIN_P2P_NCHANNELS=32" "NCCL_NCHANNELS_PER_PEER=8" "NCCL_P2P_NVL_CHUNKSIZE=2097152 NCCL_MIN_P2P_NCHANNELS=32" "NCCL_P2P_USE_CUDA_MEMCPY=1"; do
  env $cfg timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/nccl_p2p_bw.py 2>/dev/null | grep GB/s | sed "s|^|[$cfg] |"
done
