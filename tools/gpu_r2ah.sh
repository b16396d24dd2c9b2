cd $GRAFT_REPO_ROOT
for m in 0 1 4 5 6 7; do echo "== mode $m"; ./tools/decode_trace 64 $m 2>&1 | grep -E "^CTA 0|MMA issued|converted|rep 3"; done
for m in 0 4 5 7; do echo "== T=1 mode $m"; ./tools/decode_trace 1 $m 2>&1 | grep -E "^CTA 0|converted|rep 3"; done
