B="python bench.py --no-cpu-baseline --sweep 0 --c3 0 --table1 0 --c4 0 --ablation 0"
for i in 1 2; do
  TACTIC_NO_SAMPLE_PREFETCH=1 $B > gpurun_out/ab2_base$i.log 2>&1
  $B > gpurun_out/ab2_pf$i.log 2>&1
done
python tools/phase_timing.py > gpurun_out/ab2_phase.log 2>&1
