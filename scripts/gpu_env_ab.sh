# Bench A/B over environment settings: ENVS="A=1 B=2;C=3" (';'-separated sets, first = baseline "").
mkdir -p gpurun_out
T=${TAG:-env}
i=0
IFS=';' read -ra SETS <<< "${ENVS}"
for set in "" "${SETS[@]}"; do
  env $set python bench.py --no-cpu-baseline --no-ablation ${BENCH_ARGS} > gpurun_out/${T}_$i.log 2>&1
  echo "$i [$set] rc=$?" >> gpurun_out/${T}_status.txt
  i=$((i+1))
done
for set in "" "${SETS[@]}"; do
  env $set python bench.py --no-cpu-baseline --no-ablation ${BENCH_ARGS} > gpurun_out/${T}_r$i.log 2>&1
  echo "r$i [$set] rc=$?" >> gpurun_out/${T}_status.txt
  i=$((i+1))
done
