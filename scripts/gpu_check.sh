# GPU check of the current tree: gpu parity tests, the default bench line, the reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/c_gpu_tests.log 2>&1; echo gputests=$? > gpurun_out/c_status.txt
python bench.py > gpurun_out/c_bench.log 2>gpurun_out/c_bench.err; echo bench=$? >> gpurun_out/c_status.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c_bench_ref.log 2>&1; echo ref=$? >> gpurun_out/c_status.txt
