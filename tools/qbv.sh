# build variants (GEM_NVCC_EXTRA defines) and bench each: bash tools/qbv.sh "-DA=1" "-DB=2 -DC=3" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "$@"; do
  GEM_NVCC_EXTRA="$v" python -c "from paper_2509_25075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-volume ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), {k:round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})"
done
