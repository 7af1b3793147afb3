# usage: K=<kernel regex> SKIP=<n> OUT=<name> ARGS="<probe args>" bash scripts/_cmd_ncu_k.sh
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip ${SKIP:-0} --launch-count 1 -o gpurun_out/$OUT -f python scripts/probe_ipg.py $ARGS > gpurun_out/${OUT}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_src.csv 2>&1
ls -la gpurun_out/$OUT*
