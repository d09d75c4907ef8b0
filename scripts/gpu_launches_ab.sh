# Launch lists (ncu, per-kernel durations) of the bench frame with and without deferral.
mkdir -p gpurun_out
T=${TAG:-la}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_defer.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/${T}_defer.csv > gpurun_out/${T}_defer.txt 2>&1
GSCG_NO_DEFER=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_nodefer.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/${T}_nodefer.csv > gpurun_out/${T}_nodefer.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_defer.log 2>&1
GSCG_NO_DEFER=1 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_nodefer.log 2>&1
