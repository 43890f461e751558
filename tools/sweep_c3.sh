cd $GRAFT_REPO_ROOT
run() { echo "== $*"; env "$@" python bench.py --no-cpu-baseline --no-accuracy --no-clocks --steps 4 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' step', d['ms_per_step'], 'fact', d['factorize_ms'], 'solve', d['solve_ms'], 'e2e', d['e2e']['ms_per_step'], 'relres', d.get('relres_vs_ktilde'))"; }
run HKS_NOP=1
run HKS_TRSM_NC=64
run HKS_TRSM_SINGLE_T=1
run HKS_LOOKAHEAD=1
run HKS_LU_GATHER=1
run HKS_FUSED_MAX=4
run HKS_FUSED_MAX=32
run HKS_PANEL_PB=16
run HKS_COND_START_LEVEL=5
