# A/B of the frame under env switches (bench headline line each), plus GPU parity tests.
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 1200 python -m pytest tests -m gpu -q -rs -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo gputests=$? > gpurun_out/${T}_status.txt
python bench.py --no-cpu-baseline > gpurun_out/${T}_base.log 2>&1; echo base=$? >> gpurun_out/${T}_status.txt
GSCG_NO_PDL=1 python bench.py --no-cpu-baseline > gpurun_out/${T}_nopdl.log 2>&1; echo nopdl=$? >> gpurun_out/${T}_status.txt
GSCG_RASTER_ONE_PHASE=1 python bench.py --no-cpu-baseline > gpurun_out/${T}_onephase.log 2>&1; echo onephase=$? >> gpurun_out/${T}_status.txt
python bench.py --config 1 --no-cpu-baseline > gpurun_out/${T}_c1.log 2>&1; echo c1=$? >> gpurun_out/${T}_status.txt
GSCG_NO_PDL=1 python bench.py --config 1 --no-cpu-baseline > gpurun_out/${T}_c1_nopdl.log 2>&1; echo c1nopdl=$? >> gpurun_out/${T}_status.txt
