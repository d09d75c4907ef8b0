# GPU parity tests + bench lines (config 3, config 1) + a launch list.
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 1200 python -m pytest tests -m gpu -q -rs -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo gputests=$? > gpurun_out/${T}_status.txt
python bench.py --no-cpu-baseline > gpurun_out/${T}_base.log 2>&1; echo base=$? >> gpurun_out/${T}_status.txt
python bench.py --config 1 --no-cpu-baseline > gpurun_out/${T}_c1.log 2>&1; echo c1=$? >> gpurun_out/${T}_status.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
