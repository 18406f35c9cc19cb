cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "$@"; do
  eval "$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-volume" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), {k:round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})"
done
