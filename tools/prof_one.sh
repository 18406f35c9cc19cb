#!/bin/bash
# ncu --set full of one launch of kernel $K (skipping $SKIP launches), summary to gpurun_out/sum_$TAG.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-9} -c ${COUNT:-1} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep 40 > gpurun_out/sum_$TAG.txt 2>&1
python tools/ncu_stalls.py gpurun_out/prof_$TAG.ncu-rep >> gpurun_out/sum_$TAG.txt 2>&1
