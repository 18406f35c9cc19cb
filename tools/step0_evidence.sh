#!/bin/bash
# Step-0 box facts and sanitizer runs -> gpurun_out/step0/ (copied to profiles/r2/)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/step0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/step0/build.log 2>&1
nvidia-smi > gpurun_out/step0/nvidia-smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/microbench tools/microbench.cu > gpurun_out/step0/microbench_build.log 2>&1 \
  && timeout 300 /tmp/microbench > gpurun_out/step0/microbench.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py > gpurun_out/step0/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/step0/sanitizer_$tool.txt
done
tail -3 gpurun_out/step0/sanitizer_*.txt
cat gpurun_out/step0/microbench.txt
