export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python scripts/ab_cfg1.py scratch_libs/lib_nosub.so paper_1810_01967_b200/libcoverblip_b200.so scratch_libs/lib_waitb.so > gpurun_out/r02g_ab.log 2>&1; echo "ab rc=$?"; tail -4 gpurun_out/r02g_ab.log
timeout 900 python -m pytest tests/test_gpu_operator_solver.py -m gpu -x -q > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02g_pytest.log
