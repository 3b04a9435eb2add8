for mb in 128 192; do for kt in "" "--no-kernel-timing"; do
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --work-mb $mb $kt 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($mb, '$kt', d['ms_per_step'], d['step_roofline']['kernel_ms_per_step'], d['phases_ms_last_step'])"
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
