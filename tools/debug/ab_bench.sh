# A/B of library env switches on the n=14 bench: prints ms/step and the pass split per setting
# usage: AB="LRE_VF3_LOGV=0 LRE_VF3_LOGV=1" bash tools/debug/ab_bench.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for kv in ${AB}; do
  for rep in 1 2; do
    env $kv timeout 300 python bench.py --n ${N:-14} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-step3 > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); w=d['whole_path']; print('$kv', round(d['ms_per_step'],3), 'p1', round(w['t_pass1_s']*1e3,3), 'p2+', round(w['t_pass2_s']*1e3,3), 'asm', round(w['t_assemble_s']*1e3,3))"
  done
done
