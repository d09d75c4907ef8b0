mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "naive or band or group" > gpurun_out/e_tests.log 2>&1; echo tests=$? > gpurun_out/e_status.txt
python bench.py --no-cpu-baseline --band-path > gpurun_out/e_bench_band.log 2>gpurun_out/e_bench_band.err; echo band=$? >> gpurun_out/e_status.txt
python bench.py --no-cpu-baseline --band-estimate > gpurun_out/e_bench_est.log 2>gpurun_out/e_bench_est.err; echo est=$? >> gpurun_out/e_status.txt
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/e_bench_c5.log 2>gpurun_out/e_bench_c5.err; echo c5=$? >> gpurun_out/e_status.txt
