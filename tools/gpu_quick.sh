#!/bin/bash
# quick iteration: build, gpu tests, bench (no cpu baseline)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?" >> gpurun_out/bench_quick.err
tail -3 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"] if d["e2e"] else None, "clocks", d["clocks"])
print("roof", d["roofline"])
for k,v in d["kernels"].items(): print(f"  {k:12s} {v['ms_per_step']*1e3:8.1f} us  {100*v['share']:5.1f}%")
PY
