# Print the bench lines of a gpu_env_ab.sh run (TAG as the argument).
T=$1
cat gpurun_out/${T}_status.txt
for f in $(ls gpurun_out/${T}_*.log | sort -V); do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split('/')[-1], d['value'], d['median_frame_ms'], d['stage_ms'], 'e2e', d['e2e']['value'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
