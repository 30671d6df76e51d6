#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the C1 smoke path (k-means build,
# decode on the oracle's clustering, dense decode) and every decode path at small sizes
# (tools/sanitize_paths.py) -- SURVEY §5.  Logs -> gpurun_out/.
#   gpurun --timeout 1800 -- 'bash tools/sanitize_c1.sh'
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool smoke rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_paths.py >> gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_paths.py cluster > gpurun_out/sanitize_cluster_$tool.log 2>&1
  echo "$tool (with the opt-in cluster decode) rc=$?" | tee -a gpurun_out/sanitize_cluster_$tool.log
done
