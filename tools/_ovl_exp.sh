# usage: CFGS="lib:ovl:workmb ..." bash tools/_ovl_exp.sh  (diagnostic A/B of the overlapped schedule)
cd $GRAFT_REPO_ROOT
b() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step']['contract'], d['step_roofline']['kernel_ms_per_step']['fft_reduce'])" 2>&1 | tail -1; }
for cfg in $CFGS; do IFS=: read lib ov wm <<< "$cfg"
  RSVD_LIB=build_var/$lib.so RSVD_OVERLAP=$ov timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --work-mb $wm > gpurun_out/ovx_${lib}_${ov}_${wm}.log 2>&1
  echo "$lib ovl=$ov work=$wm: $(b gpurun_out/ovx_${lib}_${ov}_${wm}.log)"
done
