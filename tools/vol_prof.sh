#!/bin/bash
# Volume query (row a11): parity tests, timing probe, launch list and one ncu --set full of
# k_vol_render -> gpurun_out/vol_*_$TAG
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "volume" 2>&1 | tail -3
python tools/vol_probe.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vol_launches_$TAG.csv python tools/vol_probe.py > /dev/null 2>&1
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/vol_launches_$TAG.csv")) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
d = collections.defaultdict(list)
for r in rows: d[r[4].split("(")[0][-24:]].append(float(r[-1].replace(",", "")))
for k, v in d.items(): print("%-26s %3d launches  %8.1f us" % (k, len(v), sum(v) / len(v) / 1e3))
PY
if [ -n "$FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vol_render -s 3 -c 1 -o gpurun_out/vol_prof_$TAG python tools/vol_probe.py > gpurun_out/vol_ncu_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
