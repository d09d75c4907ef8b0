mkdir -p gpurun_out
T=${TAG:-da}
for c in 1 2; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_c${c}_defer.log 2>&1
  GSCG_NO_DEFER=1 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_c${c}_nodefer.log 2>&1
done
python bench.py --no-cpu-baseline --band-estimate > gpurun_out/${T}_est_defer.log 2>&1
GSCG_NO_DEFER=1 python bench.py --no-cpu-baseline --band-estimate > gpurun_out/${T}_est_nodefer.log 2>&1
