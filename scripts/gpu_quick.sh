# Quick A/B: sort-related GPU tests (PYTEST_K), the config-3 bench line, a launch list.
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-parity or golden or sort or tie or config}" > gpurun_out/${T}_tests.log 2>&1; echo tests=$? > gpurun_out/${T}_status.txt
python bench.py --no-cpu-baseline --no-ablation > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_l.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ablation > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/${T}_l.csv > gpurun_out/${T}_l.txt 2>&1
