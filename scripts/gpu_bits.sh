# Depth-sort tag width sweep: bench stage times per GSCG_DEPTH_SORT_BITS, launch lists at two widths.
mkdir -p gpurun_out
T=${TAG:-bits}
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or golden or sort or tie or config" > gpurun_out/${T}_tests.log 2>&1; echo tests=$? > gpurun_out/${T}_status.txt
for b in 25 22 20 18; do
  GSCG_DEPTH_SORT_BITS=$b python bench.py --no-cpu-baseline --no-ablation > gpurun_out/${T}_b$b.log 2>&1; echo b$b=$? >> gpurun_out/${T}_status.txt
done
for b in 25 20; do
  GSCG_DEPTH_SORT_BITS=$b ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_l$b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ablation > /dev/null 2>&1
  python scripts/launch_table.py gpurun_out/${T}_l$b.csv > gpurun_out/${T}_l$b.txt 2>&1
done
