#!/bin/bash
# Round profile set: smoke, then ncu --set full captures of the align kernels (cold and warm L2)
# and of the precompute kernels, each after the same command ran clean without ncu.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
bash tools/gpu_prof.sh ${TAG}_align_cold > gpurun_out/${TAG}_p1.log 2>&1
bash tools/gpu_prof_warm.sh ${TAG}_align_warm > gpurun_out/${TAG}_p2.log 2>&1
bash tools/gpu_prof_pre.sh ${TAG}_pre > gpurun_out/${TAG}_p3.log 2>&1
tail -2 gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_p1.log gpurun_out/${TAG}_p2.log gpurun_out/${TAG}_p3.log | grep exit
