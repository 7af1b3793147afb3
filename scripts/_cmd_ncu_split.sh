export PYTHONPATH=.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/split_cfg1 -f python scripts/probe_split_mode.py cfg1 > gpurun_out/ncu_split_cfg1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/f16_cfg1 -f python scripts/probe_split_mode.py cfg1 > gpurun_out/ncu_f16_cfg1.log 2>&1
tail -3 gpurun_out/ncu_split_cfg1.log gpurun_out/ncu_f16_cfg1.log
