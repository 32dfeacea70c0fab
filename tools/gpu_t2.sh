cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export TRACE_REPS=1
. tools/ncu_cap.sh
cap ${CAPN:-cf_c4} ${CAPC:-4} ${CAPM:-auto} ${CAPK:-cand_flat} ${CAPS:-5}
