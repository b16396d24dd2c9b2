cd $GRAFT_REPO_ROOT
for b in prologue_trace prologue_trace_c8 prologue_trace prologue_trace_c8; do for tk in "4096 4096" "2048 4096"; do echo "== $b $tk"; ./bench/micro/$b $tk 1 2>&1 | grep -E "rep 2|CTAs traced|slot  [234]"; done; done
