export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 4 --launch-count 4 -o gpurun_out/ab_cfg1 -f python scripts/ab_cfg1.py scratch_libs/lib_old.so paper_1810_01967_b200/libcoverblip_b200.so > gpurun_out/ab_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ab_cfg1.ncu-rep --page raw --csv > gpurun_out/ab_cfg1_raw.csv 2>&1
ncu -i gpurun_out/ab_cfg1.ncu-rep --page source --csv --print-source sass > gpurun_out/ab_cfg1_src.csv 2>&1
ls -la gpurun_out/ab_cfg1*
