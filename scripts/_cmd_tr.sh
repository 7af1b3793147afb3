export PYTHONPATH=.
L=paper_1810_01967_b200
echo "== trace full"; CBB_TC_DUAL=0 timeout 120 python scripts/trace_tc.py 2>&1 | tail -24
echo "== trace empty"; CBB_TC_DUAL=0 CBB_LIB_PATH=$L/libcoverblip_b200_trace_empty.so timeout 120 python scripts/trace_tc.py 2>&1 | tail -24
