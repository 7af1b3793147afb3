# launch list (gpu__time_duration) of the host-driven cfg4 / cfg2 IPG loops: per-kernel shares
export PYTHONPATH=.
mkdir -p gpurun_out
R=${R:-r02h}
for cfg in cfg4 cfg2; do
IT=20; [ $cfg = cfg2 ] && IT=22
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ipg_${cfg}_launches_$R.csv python scripts/probe_ipg.py $cfg $IT nograph > gpurun_out/ipg_${cfg}_$R.log 2>&1
echo "ncu $cfg rc=$?"; tail -25 gpurun_out/ipg_${cfg}_$R.log | head -3
python scripts/summarize_ncu.py launches gpurun_out/ipg_${cfg}_launches_$R.csv gpurun_out/ipg_${cfg}_${IT}it_hostloop_launches_summary_$R.txt "ncu --metrics gpu__time_duration.sum --profile-from-start off python scripts/probe_ipg.py $cfg $IT nograph ($IT host-driven IPG iterations)" | head -32
done
rm -f gpurun_out/*.csv
