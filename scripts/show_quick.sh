# Print the tests, bench line and launch list of a gpu_quick.sh run (TAG as the argument).
T=$1
cat gpurun_out/${T}_status.txt; tail -1 gpurun_out/${T}_tests.log
python - $T <<'PY'
import json,sys
d=json.loads(open(f'/root/repo/gpurun_out/{sys.argv[1]}_bench.log').read().strip().splitlines()[-1])
print(d['value'], d['median_frame_ms'], d['stage_ms'], 'e2e', d['e2e']['value'])
PY
grep -v "k_set_power\|k_copy_seg\|at::" gpurun_out/${T}_l.txt
