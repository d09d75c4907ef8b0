# Quick GPU check of a kernel change: gpu parity tests, the default bench line, a launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_gpu_tests.log 2>&1; echo gputests=$? > gpurun_out/q_status.txt
python bench.py --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo bench=$? >> gpurun_out/q_status.txt
python bench.py --config 4 --no-cpu-baseline > gpurun_out/q_bench_c4.log 2>&1; echo c4=$? >> gpurun_out/q_status.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1; echo launches=$? >> gpurun_out/q_status.txt
python scripts/launch_table.py gpurun_out/q_launches.csv > gpurun_out/q_launches.txt 2>&1
