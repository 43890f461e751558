cd $GRAFT_REPO_ROOT
CFG=${CFG:-C3}
run() { echo "== $*"; env "$@" python bench.py --config $CFG --no-cpu-baseline --no-accuracy --no-clocks --steps 4 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' step', d['ms_per_step'], 'fact', d['factorize_ms'], 'solve', d['solve_ms'], 'e2e', d['e2e']['ms_per_step'], 'relres', d.get('relres_vs_ktilde'))"; }
for v in "$@"; do run $v; done
