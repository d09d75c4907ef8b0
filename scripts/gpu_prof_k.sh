# ncu --set full of selected kernels of one clean config-3 frame: KREGEX (ncu -k regex), TAG.
mkdir -p gpurun_out
T=${TAG:-pk}
ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:${KREGEX}" -o /tmp/prof_${T} python scripts/profile_frame.py --frames 1 --warmup 2 > gpurun_out/${T}_ncu.log 2>&1; echo full=$? > gpurun_out/${T}_status.txt
python scripts/ncu_summary.py /tmp/prof_${T}.ncu-rep > gpurun_out/${T}_summary.txt 2>&1
ncu -i /tmp/prof_${T}.ncu-rep --page details > gpurun_out/${T}_details.txt 2>&1
for k in ${KLIST}; do python scripts/ncu_source_top.py /tmp/prof_${T}.ncu-rep $k > gpurun_out/${T}_source_$k.txt 2>&1; done
