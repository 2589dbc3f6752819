# per-kernel ncu times (regex $KREGEX) of one bench run per library variant
L=paper_2011_12895_b200/_lib
cp $L/libtlg_b200.so /tmp/libtlg_b200.keep.so
for v in ${VARIANTS:-cur}; do
  cp $L/variants/lib_$v.so $L/libtlg_b200.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-loss}" --csv --log-file gpurun_out/kt_$v.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer > /dev/null 2>&1
  python3 - <<PY
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/kt_$v.csv")) if len(r)>10]
h=rows[0]; k=h.index("Kernel Name"); m=h.index("Metric Value")
agg=collections.defaultdict(list)
for r in rows[1:]: agg[r[k].split("(")[0][-40:]].append(float(r[m]))
print("$v", {n: round(sum(x)/len(x)/1e3,1) for n,x in agg.items()})
PY
done
cp /tmp/libtlg_b200.keep.so $L/libtlg_b200.so
