export PYTHONPATH=.
for c in 1 2 4; do CBB_TC_CLUSTER=$c timeout 120 python scripts/probe_mfk.py 2>&1 | tail -1 | sed "s/^/csz=$c /"; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CBB_TC_CLUSTER=4 timeout 600 python -m pytest tests/test_gpu_projection.py tests/test_gpu_split.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -3
