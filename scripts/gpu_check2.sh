mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "band or group or expf or oom or past" > gpurun_out/d_tests.log 2>&1; echo tests=$? > gpurun_out/d_status.txt
python bench.py --no-cpu-baseline > gpurun_out/d_bench.log 2>gpurun_out/d_bench.err; echo bench=$? >> gpurun_out/d_status.txt
python bench.py --no-cpu-baseline --band-path > gpurun_out/d_bench_band.log 2>gpurun_out/d_bench_band.err; echo band=$? >> gpurun_out/d_status.txt
python scripts/band_estimate.py > gpurun_out/d_band_est.log 2>&1; echo est=$? >> gpurun_out/d_status.txt
