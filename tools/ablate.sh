#!/bin/bash
# Ablation runs (experiments only, never the product): rebuild libgem.so from
# paper_2509_25075_b200/csrc/render_abl.cu.txt with each '|'-separated flag set in ABL_FLAGS and
# print the per-kernel times of the kernels matching KSEL; restores render.cu afterwards.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_2509_25075_b200/csrc/render.cu /tmp/render_orig.cu
IFS='|' read -ra SETS <<< "${ABL_FLAGS}"
for F in "" "${SETS[@]}"; do
  cp paper_2509_25075_b200/csrc/render_abl.cu.txt paper_2509_25075_b200/csrc/render.cu
  GEM_EXTRA_FLAGS="$F" python -c "
import os
from paper_2509_25075_b200 import build as b
b.NVCC_FLAGS += os.environ['GEM_EXTRA_FLAGS'].split()
b.build(force=True)" > /dev/null 2>&1
  echo "== [$F]"
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items() if '$KSEL' in k})"
done
cp /tmp/render_orig.cu paper_2509_25075_b200/csrc/render.cu
