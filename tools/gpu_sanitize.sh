cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r02}_sanitizer.txt; : > $O
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/debug/sanitize_smoke.py" >> $O
  timeout 1500 compute-sanitizer --tool $tool python tools/debug/sanitize_smoke.py 2>&1 | grep -v "^=========     \|^========= Program hit\|Saved host backtrace" | tail -5 >> $O
done
cat $O
