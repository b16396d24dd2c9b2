cd $GRAFT_REPO_ROOT
for b in decode_trace decode_trace_bulk decode_trace decode_trace_bulk; do for t in 64 1; do echo "== $b T=$t"; ./tools/$b $t 0 2>&1 | grep -E "rep 3|^CTA 0: start 0.00 "; ./tools/$b $t 2 2>&1 | grep -E "rep 3|^CTA 0: start 1"; done; done
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x 2>&1 | tail -2
