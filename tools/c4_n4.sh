# 4-GPU checks: the native store's golden blobs + the mixed lazy reshard at N=4, C4 at N=4 (bench.py + C++ host)
timeout 600 python -m pytest tests/test_reshard.py -m gpu -q -p no:cacheprovider -k "dstore or mixed" > gpurun_out/r02_gpu_n4_reshard.log 2>&1; echo EXIT $? >> gpurun_out/r02_gpu_n4_reshard.log
tail -3 gpurun_out/r02_gpu_n4_reshard.log
for tr in pull nccl; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c4 --gpus 4 --transport $tr --steps 50 --warmup 5 2>/dev/null | tail -1 > gpurun_out/r02_c4_n4_$tr.json
python -c "import json; d=json.load(open('gpurun_out/r02_c4_n4_$tr.json')); print('$tr', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
done
DFX_DSTORE_TRACE=1 timeout 120 ./cpp/_build/bench_dstore 4 50 5 pull 2>&1 | grep -v "rank [123]" | cut -c1-300
