export PYTHONPATH=.
mkdir -p gpurun_out
R=${R:-r01h}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_${R}_reference.json 2> gpurun_out/bench_${R}_reference.err
echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches_$R.csv python bench.py --steps 3 --warmup 3 --skip-cfg3 > gpurun_out/ncu_launch_$R.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/prof_bench_$R -f python bench.py --skip-cfg2 --skip-cfg3 --skip-cfg4 > gpurun_out/ncu_full_$R.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/prof_bench_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$R.csv 2>&1
ls -la gpurun_out | tail -12
