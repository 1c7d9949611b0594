cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/e2e_breakdown.py cfg4 2>&1 | tail -6
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
