# sub-stage fp16 screen A/B + spin variants; new tiled gather / kspace kernels: tests and operator probe
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_edges.py tests/test_gpu_split.py tests/test_gpu_operator_solver.py -m gpu -x -q > gpurun_out/r02f_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02f_pytest.log
timeout 600 python scripts/ab_cfg1.py scratch_libs/lib_nosub.so paper_1810_01967_b200/libcoverblip_b200.so scratch_libs/lib_issspin_sub.so scratch_libs/lib_epispin_sub.so scratch_libs/lib_bothspin_sub.so scratch_libs/lib_issspin.so scratch_libs/lib_epispin.so scratch_libs/lib_noslow.so > gpurun_out/r02f_ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/r02f_ab.log | tail -10
timeout 600 python scripts/probe_op.py cfg4 > gpurun_out/r02f_op_cfg4.log 2>&1; tail -2 gpurun_out/r02f_op_cfg4.log
timeout 600 python scripts/probe_op.py cfg2 > gpurun_out/r02f_op_cfg2.log 2>&1; tail -2 gpurun_out/r02f_op_cfg2.log
