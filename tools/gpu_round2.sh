#!/bin/bash
# Round-2 evidence session: GPU tests, smoke, bench line (+ oracle cpu_baseline), reference arm,
# ncu launch list of the bench command, --set full captures of the step's main kernels and of the
# measured TMA variants.  Everything under gpurun_out/round2/ (summaries copied to profiles/r2/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r2f}
O=gpurun_out/round2
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?" >> $O/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-volume"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_$TAG.csv $CMD > $O/ncu_launch.log 2>&1
python tools/launch_share.py $O/launches_$TAG.csv k_prep > $O/launches_${TAG}_last_step_share.txt 2>&1
# one launch each of the main kernels in a timed step (skip the ring generation and warm-up)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_render_fwd|k_render_bwd|k_splat|k_fill|k_ctf_colspec|k_scan_pp" -s 27 -c 6 -o $O/full_$TAG $CMD > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/full_$TAG.ncu-rep 40 > $O/ncu_full_summary_$TAG.txt 2>&1
python tools/ncu_stalls.py $O/full_$TAG.ncu-rep >> $O/ncu_full_summary_$TAG.txt 2>&1
for k in k_render_fwd_le k_render_bwd k_splat_count k_fill k_ctf_colspec; do
  python tools/ncu_lines.py $O/full_$TAG.ncu-rep $k 50 > $O/ncu_lines_${k}_$TAG.txt 2>&1
done
# TMA variants (measured, not kept): backward record staging by cp.async.bulk + mbarrier,
# forward bulk L2 prefetch of the next particles' records
for v in "-DGEM_BWD_TMA=1:k_render_bwd:bwd_tma" "-DGEM_FWD_L2PF=2:k_render_fwd:fwd_l2pf"; do
  IFS=: read defs kre name <<< "$v"
  GEM_NVCC_EXTRA="$defs" python -c "from paper_2509_25075_b200 import build as b; b.build(force=True)" > $O/build_$name.log 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-volume > $O/bench_$name.json 2>/dev/null
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 5 -c 1 -o $O/full_$name $CMD > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py $O/full_$name.ncu-rep 30 > $O/ncu_full_summary_$name.txt 2>&1
  python tools/ncu_stalls.py $O/full_$name.ncu-rep >> $O/ncu_full_summary_$name.txt 2>&1
done
python -c "from paper_2509_25075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
# other workloads and batch sizes (no cpu baseline / e2e): S, P and the batch sweep at R
for a in "--config S" "--config P" "--batch 128" "--batch 512" "--state init"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-volume $a > "$O/bench_$(echo $a | tr -d ' -')_$TAG.json" 2>/dev/null
done
# the volume query's launch list and one --set full capture of its render kernel
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/vol_launches_$TAG.csv python tools/vol_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vol_render|k_vol_stage" -s 6 -c 2 -o $O/full_vol_$TAG python tools/vol_probe.py > $O/ncu_vol.log 2>&1
python tools/ncu_summary.py $O/full_vol_$TAG.ncu-rep 30 > $O/ncu_full_summary_vol_$TAG.txt 2>&1
python tools/ncu_stalls.py $O/full_vol_$TAG.ncu-rep >> $O/ncu_full_summary_vol_$TAG.txt 2>&1
# the e2e path: PCIe bandwidth and copy/compute interference
python tools/h2d_bw.py > $O/h2d_bw_$TAG.txt 2>&1
python tools/copy_interference.py > $O/copy_interference_$TAG.txt 2>&1
tail -2 $O/pytest_gpu.log; tail -2 $O/smoke.log; tail -1 $O/bench_$TAG.err
