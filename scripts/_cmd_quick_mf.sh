# quick A/B of the fp16 screen: kernel time on cfg1 + projection parity tests
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 120 python scripts/probe_mfk.py 2>&1 | tail -1
timeout 120 python scripts/probe_mfk.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_projection.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -2
