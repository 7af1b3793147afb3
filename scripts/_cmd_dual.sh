export PYTHONPATH=.
L=paper_1810_01967_b200
for p in 0 1; do CBB_TC_DUAL=$p timeout 100 python scripts/probe_mfk.py 2>&1 | tail -1 | sed "s/^/dual=$p /"; done
for p in 0 1; do CBB_TC_DUAL=$p CBB_LIB_PATH=$L/libcoverblip_b200_EMPTY.so timeout 100 python scripts/probe_mfk.py 2>&1 | tail -1 | sed "s/^/EMPTY dual=$p /"; done
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
