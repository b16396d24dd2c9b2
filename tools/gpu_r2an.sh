cd $GRAFT_REPO_ROOT
for b in prologue_trace prologue_trace_f2f prologue_trace prologue_trace_f2f; do for tk in "4096 4096" "2048 4096"; do echo "== $b $tk"; ./bench/micro/$b $tk 1 2>&1 | grep -E "rep 2|slot  [234]"; done; done
