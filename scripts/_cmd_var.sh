export PYTHONPATH=.
L=paper_1810_01967_b200
for v in "" _EMPTY; do CBB_LIB_PATH=$L/libcoverblip_b200$v.so timeout 100 python scripts/probe_mfk.py 2>&1 | tail -1; done
timeout 100 python scripts/probe_split_mode.py coh coh20 2>&1 | grep "tcgen05_split "
echo "== trace full"; timeout 120 python scripts/trace_tc.py 2>&1 | grep -v "voxel tile" | tail -18
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
