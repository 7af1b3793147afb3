export PYTHONPATH=.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err
echo "bench rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches_r01g.csv python bench.py > gpurun_out/ncu_launch_r01g.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/prof_bench_r01g -f python bench.py --skip-cfg2 --skip-cfg3 --skip-cfg4 > gpurun_out/ncu_full_r01g.log 2>&1
echo "ncu full rc=$?"
