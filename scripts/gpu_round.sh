# One GPU round: smoke, gpu tests, bench lines, launch list, one ncu --set full capture.
# Reports are summarised on the box and the .ncu-rep removed (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo gputests=$? >> gpurun_out/status.txt
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status.txt
for c in 1 2 4 5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo c$c=$? >> gpurun_out/status.txt; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v6.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/status.txt
python scripts/launch_table.py gpurun_out/launches_v6.csv > gpurun_out/launches_v6.txt 2>&1
ncu --set full --clock-control none --import-source on -o /tmp/prof_full7 python scripts/profile_frame.py --frames 1 > gpurun_out/ncu_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
python scripts/ncu_summary.py /tmp/prof_full7.ncu-rep gpurun_out/ncu_summary.json > gpurun_out/ncu_full_v6.txt 2>&1
for k in k_sort_downsweep k_sort_upsweep k_emit_scatter k_raster16q k_project k_cell_fixup; do
  python scripts/ncu_source_top.py /tmp/prof_full7.ncu-rep $k > gpurun_out/source_$k.txt 2>&1
done
ls -la gpurun_out >> gpurun_out/status.txt
