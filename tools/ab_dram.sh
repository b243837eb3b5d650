cd $GRAFT_REPO_ROOT
for v in pf1 pf0; do
  SVX_LIB_PATH=$PWD/variants/libsvx_$v.so ncu --cache-control none --clock-control none -k regex:"k_(resolve|update_slots)" --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --log-file gpurun_out/dram_$v.csv python bench.py --steps 3 --warmup 3 --profile-frames 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/dram_$v.csv")))
h=[i for i,r in enumerate(rows) if "Metric Name" in r][0]; hdr=rows[h]
from collections import defaultdict
agg=defaultdict(lambda: defaultdict(list))
for r in rows[h+1:]:
    k=r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
    agg[k][r[hdr.index("Metric Name")]].append(float(r[hdr.index("Metric Value")].replace(",","")))
for k,m in agg.items():
    print("$v", k, {n: round(sum(v[-3:])/3/1e6,2) if "bytes" in n else round(sum(v[-3:])/3/1e3,1) for n,v in m.items()})
PY
done
bash tools/ab_variants.sh
