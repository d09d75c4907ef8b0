# compute-sanitizer over one BASELINE config-1 frame (100 K splats, 512x512) after a warm-up
# frame: memcheck (out-of-bounds / misaligned accesses, device-side), racecheck (shared
# memory hazards in the warp-synchronous sort / raster kernels) and synccheck.
mkdir -p gpurun_out
T=${TAG:-san}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python scripts/profile_frame.py --config 1 --frames 1 --warmup 1 > gpurun_out/${T}_$tool.log 2>&1
  echo $tool=$? >> gpurun_out/${T}_status.txt
done
