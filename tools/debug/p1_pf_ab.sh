# A/B of pass-1 L2-prefetch variants (alternative builds under paper_1602_08604_b200/_lib_<name>)
B="python bench.py --qubits ${N:-14} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-step3"
ext() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); w=d['whole_path']; print(sys.argv[1], round(d['ms_per_step'],3), 'pass1', round(w['t_pass1_s']*1e3,3))" "$1"; }
for r in 1 2 3; do
  timeout 300 $B 2>/dev/null | ext default
  for V in ${VARIANTS:-pfe}; do
    LRE_LIB_PATH=$PWD/paper_1602_08604_b200/_lib_$V/liblre_b200.so timeout 300 $B 2>/dev/null | ext $V
  done
done
