# ad-hoc GPU batch: selected gpu tests + short bench + ncu launch list (logs in gpurun_out/)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
TAG=${TAG:-x}
if [ -z "$SKIP_TESTS" ]; then
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 ${PYTEST_SEL:+-k "$PYTEST_SEL"} > $O/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$TAG.log
tail -25 $O/pytest_$TAG.log
fi
for n in ${BENCH_NS:-14}; do
timeout 600 python bench.py --n $n --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-step3 > $O/bench_${TAG}_n$n.json 2> $O/bench_${TAG}_n$n.err
echo "bench n=$n rc=$?"; cat $O/bench_${TAG}_n$n.json | head -c 1500; echo; tail -3 $O/bench_${TAG}_n$n.err
done
if [ -n "$NCU_N" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_${TAG}_n$NCU_N.csv python bench.py --n $NCU_N --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
fi
if [ -n "$NCU_FULL" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$NCU_FULL -s ${NCU_SKIP:-1} -c 1 \
    -o $O/full_${TAG}_$NCU_FULL -f python bench.py --n ${NCU_FULL_N:-14} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > $O/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
fi
