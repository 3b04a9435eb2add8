#!/bin/bash
# Workspace-size sweep of the Large step: headline ms/step, align phase, per-kernel ms (event pass).
for mb in ${@:-64 128}; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --work-mb $mb 2>/dev/null | tail -1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read()); print($mb, d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'])"
done
