# ncu --set full of the cfg1 fp16 screen with per-SASS-line execution counts (source page)
export PYTHONPATH=.
mkdir -p gpurun_out
OUT=${OUT:-r02e_mf}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/$OUT -f python scripts/probe_mfk.py > gpurun_out/${OUT}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${OUT}_ncu.log
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_src.csv 2>&1
ls -la gpurun_out/$OUT*
