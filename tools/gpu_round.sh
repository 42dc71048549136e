#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, reference bench, ncu launch list
# + `ncu --set full` captures of the top kernels (bench + the C4 long-trace path).
# usage (from the repo root, under gpurun):  bash tools/gpu_round.sh TAG
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $OUT/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 > $OUT/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4_$TAG.csv \
    python tools/c4_breakdown.py > $OUT/ncu_launch_c4_$TAG.log 2>&1
for K in k_cand_step k_replay_warp k_form_models k_merge_batches_warp k_merge_arrivals_scen k_noise_table k_gen_arrivals k_slo k_features k_scen_stats k_scen_solve k_scen_qr k_scen_finish k_rls_g8 k_eval_warp k_score_decisions_lane k_dispatch_sets k_sgd k_ols_partial k_ols_windows_tma k_cand_step_host; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/prof_${TAG}_$K \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 > $OUT/ncu_${TAG}_$K.log 2>&1
done
for K in k_bin_runs k_bin_classify k_gen_gaps k_form_chunks k_arr_place k_bat_place k_jobs_replay k_jobs_verify_big k_slo_big_hist; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/prof_${TAG}_$K \
    python tools/c4_breakdown.py > $OUT/ncu_${TAG}_$K.log 2>&1
done

# summarise on the box (ncu is there) and keep gpurun_out under the 64 MiB copy-back limit
python tools/ncu_summary.py $TAG $OUT/prof_${TAG}_*.ncu-rep --launches $OUT/launches_$TAG.csv > $OUT/summary_$TAG.log 2>&1
ncu -i $OUT/prof_${TAG}_k_cand_step.ncu-rep --page raw --csv > $OUT/raw_k_cand_step_$TAG.csv 2>/dev/null
cp profiles/ncu_$TAG.md profiles/ncu_summary.json $OUT/ 2>/dev/null

find $OUT -name "prof_${TAG}_*.ncu-rep" ! -name "prof_${TAG}_k_cand_step.ncu-rep" ! -name "prof_${TAG}_k_replay_warp.ncu-rep" ! -name "prof_${TAG}_k_bin_runs.ncu-rep" ! -name "prof_${TAG}_k_ols_windows_tma.ncu-rep" -delete
du -sh $OUT
echo done
