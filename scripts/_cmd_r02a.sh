export PYTHONPATH=.
mkdir -p gpurun_out
L=paper_1810_01967_b200
echo "== normal"; timeout 120 python scripts/probe_cfg1.py 2>&1 | tail -3
echo "== empty epilogue"; CBB_LIB_PATH=$L/libcoverblip_b200_empty.so timeout 120 python scripts/probe_cfg1.py 2>&1 | tail -3
echo "== trace"; timeout 120 python scripts/trace_tc.py 2>&1 | tail -25
timeout 600 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/src_cfg1 -f python scripts/probe_cfg1.py > gpurun_out/ncu_src.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/src_cfg1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_cfg1_sass.csv 2>&1
echo "export rc=$?"; ls -la gpurun_out
