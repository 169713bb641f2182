# C3 under ncu: GAE parity per scan variant, launch lists of the fused pass and of the two-launch step, one full
# capture of each scan kernel (seg: dfx_gae's default; lb: the fused pass's)
for v in seg lb; do DFX_GAE_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sweep.py -q -x -k "gae or c3" -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -8; done
for v in seg lb; do
  DFX_GAE_VARIANT=$v python tools/c3_prof.py --fused >/dev/null 2>&1 && DFX_GAE_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3f_launch_$v.csv python tools/c3_prof.py --fused > /dev/null 2>&1
  DFX_GAE_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launch_$v.csv python tools/c3_prof.py > /dev/null 2>&1
done
DFX_GAE_VARIANT=lb timeout 600 ncu --set full --clock-control none --import-source on -k regex:gae_smem -s 2 -c 1 -o gpurun_out/prof_c3f_lb python tools/c3_prof.py --fused > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gae_seg -s 2 -c 1 -o gpurun_out/prof_c3_seg python tools/c3_prof.py > /dev/null 2>&1
ls gpurun_out
