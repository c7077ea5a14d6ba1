#!/bin/bash
# One GPU session collecting the round's evidence (logs in gpurun_out/, tag $TAG):
# smoke, the full -m gpu suite, both bench arms at n=14, bench n=12, the distributed
# arm at world 1, the ncu launch list at n=14 and --set full captures of the step-(ii)
# and final-pass kernels.  Each step is bounded by its own timeout.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O; T=${TAG:-r02}
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > $O/${T}_gpu_info.txt 2>&1
nproc >> $O/${T}_gpu_info.txt; free -g >> $O/${T}_gpu_info.txt; lscpu | grep "Model name" >> $O/${T}_gpu_info.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 300 python __graft_entry__.py smoke > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $O/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest_gpu.log
fi
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_bench_reference_n14.json 2> $O/${T}_bench_reference_n14.err
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_default_n14.json 2> $O/${T}_bench_default_n14.err
timeout 600 python bench.py --qubits 12 --steps 20 --warmup 5 > $O/${T}_bench_n12.json 2> $O/${T}_bench_n12.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 1 --force-dist --qubits 14 --steps 10 --warmup 3 --no-e2e > $O/${T}_bench_dist_world1_n14.json 2> $O/${T}_bench_dist_world1_n14.err
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/${T}_launches_n14.csv python bench.py --qubits 14 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/${T}_ncu_launches.log 2>&1
  for k in ${NCU_KERNELS:-assemble_x8 final_mm tile_pass}; do
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/${T}_full_n14_$k -f python bench.py --qubits 14 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/${T}_ncu_full_$k.log 2>&1
    # summaries travel back; the reports (tens of MB each) only with KEEP_REP=1
    python tools/ncu_summary.py $O/${T}_full_n14_$k.ncu-rep > $O/${T}_ncu_full_n14_$k.txt 2>&1
    python tools/ncu_lines.py $O/${T}_full_n14_$k.ncu-rep 30 > $O/${T}_ncu_lines_n14_$k.txt 2>&1
    [ -n "$KEEP_REP" ] || rm -f $O/${T}_full_n14_$k.ncu-rep
  done
fi
tail -2 $O/${T}_smoke.log $O/${T}_pytest_gpu.log 2>/dev/null
for f in $O/${T}_bench_*.json; do echo "== $f"; tail -c 400 $f; echo; done
