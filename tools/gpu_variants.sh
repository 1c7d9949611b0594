cd $GRAFT_REPO_ROOT
for v in base variants/mb3.so; do
  if [ "$v" = base ]; then unset SFB_LIB; else export SFB_LIB=$GRAFT_REPO_ROOT/$v; fi
  echo "== $v"
  timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python3 -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['value'], d['phase_ms_per_step']['dense_linearize'], d['roofline']['ms_per_launch'], d['final_energy'])"
done
