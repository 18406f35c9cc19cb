#!/bin/bash
# ncu --set full of the step's main kernels (one launch each, steady state) -> gpurun_out/prof_$TAG.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-volume ${BENCH_ARGS}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_render_fwd|k_render_bwd|k_splat|k_fill|k_ctf_colspec}" -s ${SKIP:-12} -c ${COUNT:-5} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
