export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_tile|kspace_s|channels_kernel|combine_s" --launch-count 4 -o gpurun_out/op_cfg4 -f python scripts/probe_op.py cfg4 > gpurun_out/op_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/op_cfg4.ncu-rep --page details --csv > gpurun_out/op_cfg4_details.csv 2>&1
ncu -i gpurun_out/op_cfg4.ncu-rep --page source --csv --print-source sass > gpurun_out/op_cfg4_src.csv 2>&1
ls -la gpurun_out/op_cfg4*
