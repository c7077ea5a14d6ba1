B="python bench.py --qubits 14 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-step3"
ext() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); w=d['whole_path']; print(sys.argv[1], round(d['ms_per_step'],3), 'pass1', round(w['t_pass1_s']*1e3,3))" "$1"; }
for r in 1 2; do
  timeout 300 $B 2>/dev/null | ext default
  LRE_P1_SYNC=bar timeout 300 $B 2>/dev/null | ext bar
done
