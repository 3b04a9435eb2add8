export CUDA_LAUNCH_BLOCKING=1
for args in "512 256 64 256 16 pair" "512 256 64 256 16 image" "512 256 64 256 16 land" "64 256 64 256 16 land" "32 256 64 256 16 land" "512 256 128 512 24 land" "512 256 32 128 8 land" "512 256 32 64 8 land"; do
 echo "== $args"; timeout 120 python tools/repro_land.py $args 2>&1 | tail -1
done
