#!/bin/bash
# One GPU round trip: gpu tests, bench, launch list + one ncu --set full capture of the streaming kernel.
# usage (on the box): bash tools/gpu_cycle.sh TAG [KERNEL_REGEX] [PROF_ARGS]
TAG=${1:-run}; KRE=${2:-loss_slots}; PARGS=${3:-"--steps 2"}
mkdir -p gpurun_out
python paper_2507_13833_b200/build.py > /dev/null || exit 1  # never measure a stale libdfx.so
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo bench_exit=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]);print('value',d['value'],'ms',d['ms_per_step'],'roof',d['roofline']['frac'],d['roofline']['kernel_ms'],'e2e',d['e2e']['value'] if d.get('e2e') else None,'clk',d['clocks'])" 2>&1 | tail -2
timeout 120 python tools/prof_step.py $PARGS > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py $PARGS > gpurun_out/ncu1_$TAG.log 2>&1
echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/prof_$TAG python tools/prof_step.py $PARGS > gpurun_out/ncu2_$TAG.log 2>&1
echo ncu2=$?
