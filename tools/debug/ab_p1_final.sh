# final check of the pass-1 configuration: default vs lockstep barrier (LRE_P1_SYNC=bar) vs prefetch 3 steps ahead (-DLRE_PF3 build in _lib_pf3)
B="python bench.py --qubits 14 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-step3"
ext() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); w=d['whole_path']; print(sys.argv[1], round(d['ms_per_step'],3), 'p1', round(w['t_pass1_s']*1e3,3))" "$1"; }
for r in 1 2 3; do
  timeout 300 $B 2>/dev/null | ext default
  LRE_P1_SYNC=bar timeout 300 $B 2>/dev/null | ext bar
  LRE_LIB_PATH=$PWD/paper_1602_08604_b200/_lib_pf3/liblre_b200.so timeout 300 $B 2>/dev/null | ext pf3
done
