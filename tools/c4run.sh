# C4 round trip on the box (N = the GPUs given to the call): pytest of the native store, bench.py --workload c4
# (Python mirror over the C ABI), and cpp/bench_dstore (the C++ host, fork per GPU), both transports.
N=${N:-2}
timeout 600 python -m pytest tests/test_reshard.py -m gpu -q -x -p no:cacheprovider -k "dstore" > gpurun_out/r02_gpu_dstore_n$N.log 2>&1; echo EXIT $? >> gpurun_out/r02_gpu_dstore_n$N.log
tail -2 gpurun_out/r02_gpu_dstore_n$N.log
timeout 120 python bench.py --workload c4 --steps 50 --warmup 5 > gpurun_out/r02_c4c_n1.json 2> gpurun_out/r02_c4c_n1.err
for tr in pull nccl; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c4 --gpus $N --transport $tr --steps 50 --warmup 5 > gpurun_out/r02_c4c_n${N}_$tr.json 2> gpurun_out/r02_c4c_n${N}_$tr.err
done
for f in gpurun_out/r02_c4c_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])")"; done
for n in 1 $N; do for tr in pull nccl; do timeout 120 ./cpp/_build/bench_dstore $n 50 5 $tr; done; done 2>&1 | tee gpurun_out/r02_cpp_dstore_n$N.log
