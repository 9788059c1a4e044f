# quick GPU check: parity tests + per-launch timing on configs 2 and 5 (n=2M)
make -C paper_2312_00538_b200/csrc >/dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for c in "2" "5 --n 2000000" "4"; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['n'], 'ms/step %.4f'%d['ms_per_step'], 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'], 'fp64frac %.3f'%d['roofline']['fp64']['frac']); print('  ', {k: round(v,4) for k,v in d['per_launch_ms'].items()})"
done
