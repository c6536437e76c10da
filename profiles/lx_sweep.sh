for lx in 10 8 9 11 13 16 5 7; do
  ST_LX=$lx python bench.py --steps 50 --no-cpu-baseline --sweep 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('Lx', $lx, round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done
