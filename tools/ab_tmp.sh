B="python bench.py --no-cpu-baseline --sweep 0 --c3 0 --table1 0 --c4 0 --ablation 0"
for i in 1 2; do
  TACTIC_LIB=$PWD/paper_2502_12216_b200/lib/libtactic_ab.so $B > gpurun_out/ab20_head$i.log 2>&1
  $B > gpurun_out/ab20_new$i.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab20_gputest.log 2>&1
