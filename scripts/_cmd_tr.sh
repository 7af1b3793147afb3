export PYTHONPATH=.
L=paper_1810_01967_b200
echo "== trace full"; timeout 120 python scripts/trace_tc.py 2>&1 | grep -v "voxel tile" | tail -18
echo "== trace empty"; CBB_LIB_PATH=$L/libcoverblip_b200_trace_empty.so timeout 120 python scripts/trace_tc.py 2>&1 | grep -v "voxel tile" | tail -18
