# Round-2 re-entry: GPU tests, then the profiling recipe (bench, reference arm, launch list, ncu full captures)
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02e_pytest.log
R=r02e bash scripts/_cmd_profiles.sh
