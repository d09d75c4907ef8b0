# One full GPU round: smoke, gpu tests, reference unit tests on the drop-in API, bench lines
# (headline + reference arm + configs 1/2/4/5 + region-split estimate), a launch list and an
# ncu --set full capture of one frame (summarised on the box; the .ncu-rep stays there).
mkdir -p gpurun_out
T=${TAG:-r02}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? > gpurun_out/${T}_status.txt
./oracle/_ref/ref_api_tests > gpurun_out/${T}_ref_api.log 2>&1; echo refapi=$? >> gpurun_out/${T}_status.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/${T}_gpu_tests.log 2>&1; echo gputests=$? >> gpurun_out/${T}_status.txt
python bench.py --band-estimate > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo bench=$? >> gpurun_out/${T}_status.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo ref=$? >> gpurun_out/${T}_status.txt
for c in 1 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_c$c.log 2>&1; echo c$c=$? >> gpurun_out/${T}_status.txt; done
timeout 1200 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/${T}_bench_c5.log 2>gpurun_out/${T}_bench_c5.err; echo c5=$? >> gpurun_out/${T}_status.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/${T}_status.txt
python scripts/launch_table.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/prof_${T} python scripts/profile_frame.py --frames 1 --warmup 2 > gpurun_out/${T}_ncu_full.log 2>&1; echo full=$? >> gpurun_out/${T}_status.txt
python scripts/ncu_summary.py /tmp/prof_${T}.ncu-rep gpurun_out/${T}_ncu_summary.json > gpurun_out/${T}_ncu_full.txt 2>&1
for k in k_raster16q k_project k_sort_downsweep k_sort_upsweep k_emit_scatter k_cell_fixup k_depth_bucket_scatter k_depth_bucket_local; do
  python scripts/ncu_source_top.py /tmp/prof_${T}.ncu-rep $k > gpurun_out/${T}_source_$k.txt 2>&1
done
ncu -i /tmp/prof_${T}.ncu-rep --page raw --csv --metrics smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,launch__registers_per_thread > gpurun_out/${T}_ncu_extra.csv 2>&1
ls -la gpurun_out >> gpurun_out/${T}_status.txt
