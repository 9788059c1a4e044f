# quick GPU check: parity tests + per-launch timing. CONFIGS is a ';'-separated list of bench args.
make -C paper_2312_00538_b200/csrc >/dev/null || exit 1
mkdir -p gpurun_out
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader
IFS=';' read -ra CFGS <<< "${CONFIGS:-2;5 --n 2000000;4}"
for c in "${CFGS[@]}"; do
  python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:5], d['config']['n'], 'ms/step %.4f'%d['ms_per_step'], 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'], 'fp64frac %.3f'%d['roofline']['fp64']['frac'], 'clk', d['clocks']['sm_mhz']); print('  ', {k: round(v,4) for k,v in d['per_launch_ms'].items()})"
done
