# ncu launch list of one config (CFG env), one lane, graphs off
cd $GRAFT_REPO_ROOT
CFG=${CFG:-cfg3}
VDAMP_GRAPHS=0 VDAMP_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_${CFG}_launches.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/launches_${CFG}_ncu.log 2>&1; echo ncu rc=$?
python - <<'P'
import csv,os,collections
cfg=os.environ.get("CFG","cfg3")
rows=[r for r in csv.reader(open(f"gpurun_out/launches_{cfg}_launches.csv")) if len(r)>5]
hdr=rows[0]; ik=hdr.index("Kernel Name"); iv=hdr.index("Metric Value"); ig=hdr.index("Grid Size"); ib=hdr.index("Block Size")
for r in rows[1:40]:
    print(r[ik][:60], r[ig], r[ib], r[iv])
P
