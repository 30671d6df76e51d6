#!/bin/bash
# One gpurun call: bench line, ncu launch list of the bench command, ncu --set full of the decode kernels.
#   gpurun --timeout 2400 -- 'bash tools/round_profile.sh r01'
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -1 gpurun_out/bench_$R.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --sweep 0 --c3 0 --table1 0 --ablation 0 --c4 0 \
  > gpurun_out/launches_$R.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"attention_kernel|score_rank|sample_kernel|fit_unit_kernel" -s 4 -c 5 \
  -o gpurun_out/full_$R -f python tools/profile_decode.py > gpurun_out/full_$R.log 2>&1
echo "full capture rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"score_kernel|score_rank|sample_kernel|fit_unit|attention_kernel" --csv \
  --log-file gpurun_out/c3_launches_$R.csv python tools/profile_c3.py > gpurun_out/c3_launches_$R.log 2>&1
echo "c3 launch list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:km_ --csv \
  --log-file gpurun_out/km_launches_$R.csv python tools/build_timing.py --layers 8 > gpurun_out/km_launches_$R.log 2>&1
echo "build launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:km_assign_tc -s 3 -c 1 \
  -o gpurun_out/km_$R -f python tools/profile_build.py > gpurun_out/km_$R.log 2>&1
echo "k-means capture rc=$?"
