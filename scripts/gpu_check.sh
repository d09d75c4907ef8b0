# GPU check of the current tree: the reference's unit tests on the drop-in API, gpu parity
# tests, the default bench line, a launch list.
mkdir -p gpurun_out
./oracle/_ref/ref_api_tests > gpurun_out/c_ref_api.log 2>&1; echo refapi=$? > gpurun_out/c_status.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/c_gpu_tests.log 2>&1; echo gputests=$? >> gpurun_out/c_status.txt
python bench.py --no-cpu-baseline > gpurun_out/c_bench.log 2>gpurun_out/c_bench.err; echo bench=$? >> gpurun_out/c_status.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c_ncu.log 2>&1; echo launches=$? >> gpurun_out/c_status.txt
python scripts/launch_table.py gpurun_out/c_launches.csv > gpurun_out/c_launches.txt 2>&1
