# ncu --set full of the s-channel operator kernels at cfg4 and cfg2 (probe_op: apply / adjoint / residual)
export PYTHONPATH=.
timeout 600 python scripts/probe_op.py cfg4 2>&1 | tail -1
timeout 600 python scripts/probe_op.py cfg2 2>&1 | tail -1
mkdir -p gpurun_out
R=${R:-r02h}
for cfg in cfg4 cfg2; do
timeout 900 ncu --set full --clock-control none -k regex:"gather_tile1|gather_loc|gather_s_kernel|kspace_s|combine_s|channels_kernel|interleave|vec_kernel|regular_fft|vector_fft" --profile-from-start off --launch-count 90 -o /tmp/prof_op_${cfg}_$R -f python scripts/probe_op.py $cfg > gpurun_out/ncu_op_${cfg}_$R.log 2>&1
echo "ncu op $cfg rc=$?"
python scripts/summarize_ncu_multi.py /tmp/prof_op_${cfg}_$R.ncu-rep gpurun_out/op_kernels_${cfg}_ncu_$R.txt "ncu --set full -k regex:<operator kernels> --profile-from-start off --launch-count 90 python scripts/probe_op.py $cfg"
done
