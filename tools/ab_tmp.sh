TACTIC_KM_UPDATE_PER_CLUSTER=1 python tools/build_timing.py --layers 4 > gpurun_out/km2_old.log 2>&1
python tools/build_timing.py --layers 4 > gpurun_out/km2_new.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:km_update --csv --log-file gpurun_out/km2_new.csv python tools/build_timing.py --layers 1 > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "kmeans or build or inertia or smoke or decode_unit or full" > gpurun_out/km2_tests.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/km2_alltests.log 2>&1
