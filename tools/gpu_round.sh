#!/bin/bash
# One GPU session producing the round's evidence: GPU tests, smoke, full bench line (with the
# oracle cpu_baseline), the reference arm, the ncu launch list of the bench command and a
# --set full capture of the two render kernels.  Logs to gpurun_out/, summaries to
# gpurun_out/round/ (copied to profiles/ by hand).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r1}
mkdir -p gpurun_out/round
nvidia-smi > gpurun_out/round/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/round/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/round/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/round/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/round/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/round/bench_$TAG.json 2> gpurun_out/round/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/round/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/bench_ref_$TAG.json 2> gpurun_out/round/bench_ref_$TAG.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-volume"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/round/launches_$TAG.csv $CMD > gpurun_out/round/ncu_launch.log 2>&1
# skip the observation generator's forwards (ring 1024 / batch) and the warm-up step
FSKIP=$(( 1024 / ${BATCH:-256} + 1 ))
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_fwd" -s $FSKIP -c 1 -o gpurun_out/round/full_$TAG $CMD > gpurun_out/round/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/round/full_$TAG.ncu-rep 40 > gpurun_out/round/ncu_full_summary_$TAG.txt 2>&1
python tools/ncu_stalls.py gpurun_out/round/full_$TAG.ncu-rep >> gpurun_out/round/ncu_full_summary_$TAG.txt 2>&1
tail -2 gpurun_out/round/pytest_gpu.log; tail -2 gpurun_out/round/smoke.log; cat gpurun_out/round/bench_$TAG.json; cat gpurun_out/round/bench_ref_$TAG.json; tail -3 gpurun_out/round/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_bwd" -s 1 -c 1 -o gpurun_out/round/full2_$TAG $CMD > gpurun_out/round/ncu_full2.log 2>&1
python tools/ncu_summary.py gpurun_out/round/full2_$TAG.ncu-rep 40 > gpurun_out/round/ncu_full2_summary_$TAG.txt 2>&1
python tools/ncu_stalls.py gpurun_out/round/full2_$TAG.ncu-rep >> gpurun_out/round/ncu_full2_summary_$TAG.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_splat_count|k_fill" -s 2 -c 2 -o gpurun_out/round/full3_$TAG $CMD > gpurun_out/round/ncu_full3.log 2>&1
python tools/ncu_summary.py gpurun_out/round/full3_$TAG.ncu-rep 40 > gpurun_out/round/ncu_full3_summary_$TAG.txt 2>&1
