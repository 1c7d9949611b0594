# Device-only bench of each variant library: VARIANTS="base nopf ..." (variants/NAME.so; "cur" = in-tree)
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-cur}; do
  if [ "$v" = cur ]; then unset SFB_LIB; else export SFB_LIB=$GRAFT_REPO_ROOT/variants/$v.so; fi
  timeout 900 python bench.py --config ${CFG:-cfg4} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python3 -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', round(d['value'],3), 'lin/launch', round(d['roofline']['ms_per_launch'],3), 'pcg us/it', round(d['pcg']['us_per_iteration'],2), d['phase_ms_per_step'], d['final_energy'])"
done
