# The profiling recipe of a round (B200_PROFILING.md): bench + reference arm, launch list of the
# bench, ncu --set full of the cfg1 screen and of a pruned split screen inside the cfg4 IPG.
export PYTHONPATH=.
mkdir -p gpurun_out
R=${R:-r02h}
timeout 1200 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${R}_reference.json 2> gpurun_out/bench_${R}_reference.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mf_tc|mf_ffma|rescore|prologue|gather|kspace|combine_s|channels|interleave|vec_kernel|scale_kernel|hint_tiles|prune_|exhaustive|reduce_stage|finish_sum|trial_|map_indices|coil_transpose|scatter_kernel|coherence|seg_table|rows_sorted|prep_|argmax_select|scaled_rows|_fft|DeviceRadixSort" --csv --log-file gpurun_out/bench_launches_$R.csv python bench.py --steps 3 --warmup 3 --skip-cfg3 --skip-cpu-reference > gpurun_out/ncu_launch_$R.log 2>&1
echo "ncu launches rc=$?"
python scripts/summarize_ncu.py launches gpurun_out/bench_launches_$R.csv gpurun_out/bench_launches_${R}_summary.txt "ncu --metrics gpu__time_duration.sum -k regex:<the library's kernels, cuFFT, CUB sort> python bench.py --steps 3 --warmup 3 --skip-cfg3 --skip-cpu-reference (the library's kernels and cuFFT; graph-replayed launches are not listed)" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_tc_kernel --launch-skip 3 --launch-count 1 -o /tmp/prof_bench_$R -f python bench.py --skip-cfg2 --skip-cfg3 --skip-cfg4 --skip-cpu-reference > gpurun_out/ncu_full_$R.log 2>&1
echo "ncu full rc=$?"
python scripts/summarize_ncu.py full /tmp/prof_bench_$R.ncu-rep gpurun_out/mf_tc_ncu_full_$R.txt gpurun_out/roofline_traffic_$R.json "ncu --set full -k regex:mf_tc_kernel --launch-skip 3 --launch-count 1 python bench.py (cfg1 screen)" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mf_tc_kernel<64, 1, 0, 1, 0>|mf_tc_kernel" --launch-skip 14 --launch-count 1 -o /tmp/prof_split_pruned_$R -f python scripts/probe_ipg.py cfg4 8 nograph > gpurun_out/ncu_split_$R.log 2>&1
echo "ncu split rc=$?"
python scripts/summarize_ncu.py full /tmp/prof_split_pruned_$R.ncu-rep gpurun_out/mf_tc_split_pruned_cfg4_ncu_full_$R.txt gpurun_out/split_traffic_$R.json "ncu --set full, launch 15 of mf_tc_kernel in probe_ipg cfg4 8 nograph (a pruned split screen, iteration ~7)" > /dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out; ls gpurun_out/*$R*
R=$R bash scripts/_cmd_opncu.sh > gpurun_out/opncu_$R.log 2>&1; echo "op ncu rc=$?"
R=$R bash scripts/_cmd_ipglist.sh > gpurun_out/ipglist_$R.log 2>&1; echo "ipg list rc=$?"
ls gpurun_out/*$R*
