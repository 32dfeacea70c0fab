cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export TRACE_REPS=1
. tools/ncu_cap.sh
cap cf_c4 4 auto cand_flat 5
