timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for v in 1 0; do RSVD_FFT_TWREG=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print($v, d['ms_per_step'], r['kernel'][:16], r['avg_launch_ms'], d.get('step_roofline'))"; done
