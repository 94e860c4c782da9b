for v in 1 0; do
F3D_LN8=$v timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"row_ln|scatter_ln_pe" --csv --log-file gpurun_out/ad_$v.csv python tools/prof_step.py > /dev/null 2>&1
echo "== LN8=$v"; python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/ad_$v.csv")))
i=[k for k,r in enumerate(rows) if r and r[0]=="ID"][0]; h=rows[i]
for r in rows[i+1:]:
    if len(r)==len(h): print(r[h.index("Kernel Name")][:40], r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
done
