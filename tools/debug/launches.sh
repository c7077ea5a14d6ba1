# ncu launch list (time + DRAM bytes) of one n=14 step; prints the last reconstruction's kernels
# usage: [ENVS="K=V ..."] bash tools/debug/launches.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
env ${ENVS:-X=1} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_dbg.csv python bench.py --n ${N:-14} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-step3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_dbg.csv")))
hdr, d = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr is None or len(r) < len(hdr):
        continue
    x = dict(zip(hdr, r))
    d.setdefault((x["ID"], x["Kernel Name"][:48]), {})[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
items = list(d.items())
start = max(i for i, (k, v) in enumerate(items) if "tile_pass" in k[1] or "vfold_kernel" in k[1] and i > 0)
for k, v in items[start - 0:start + 8]:
    t = v["gpu__time_duration.sum"] / 1e6
    print(f"{k[1]:48s} {t:7.3f} ms  R {v['dram__bytes_read.sum']/1e9:6.2f}  W {v['dram__bytes_write.sum']/1e9:6.2f}")
PY
