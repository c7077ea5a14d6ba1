#!/bin/bash
# One GPU session: smoke + parity tests + bench + ncu launch list + ncu full captures.
# Each step is bounded by its own timeout; logs land in gpurun_out/.
#   BENCH_NS="12 14"  STEPS=10  BENCH_ARGS=...   bench sizes / args
#   NCU_N=12                                     launch list (time + DRAM bytes) of bench --n NCU_N
#   NCU_FULL_N=12 NCU_KERNELS="tile_pass vfold"  one --set full capture per kernel regex
#   SKIP_TESTS=1                                 skip smoke + pytest
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,memory.used,memory.total,clocks.sm,clocks.max.sm --format=csv > $O/gpu_info.txt 2>&1
nproc >> $O/gpu_info.txt; free -g >> $O/gpu_info.txt; lscpu | grep "Model name" >> $O/gpu_info.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for n in ${BENCH_NS:-12 14}; do
  timeout ${BENCH_TIMEOUT:-900} python bench.py --n $n --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?" >> $O/bench_n$n.err
done
if [ -n "$NCU_N" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_n$NCU_N.csv python bench.py --n $NCU_N --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/ncu_bench.log 2>&1
  echo "ncu rc=$?" >> $O/ncu_bench.log
fi
if [ -n "$NCU_FULL_N" ]; then
  for k in ${NCU_KERNELS:-tile_pass}; do
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} \
      -o $O/full_n${NCU_FULL_N}_$k -f python bench.py --n $NCU_FULL_N --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/ncu_full_$k.log 2>&1
    echo "ncu full $k rc=$?" >> $O/ncu_full_$k.log
  done
fi
tail -3 $O/smoke.log 2>/dev/null; tail -5 $O/pytest_gpu.log 2>/dev/null; cat $O/bench_n*.json; for f in $O/bench_n*.err; do tail -n 3 $f; done
