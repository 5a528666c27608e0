# ncu source-level capture of the resident kernel on configs[0] (SASS page as CSV)
O=gpurun_out
R="python tools/res_profile_run.py"
$R > $O/plain_res.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o /tmp/r02_res $R > $O/ncu4.log 2>&1
python tools/ncu_summary.py /tmp/r02_res.ncu-rep > $O/r02_resident_ncu.txt 2>&1
ncu -i /tmp/r02_res.ncu-rep --page source --csv --print-source sass > /tmp/res_sass.csv 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/res_sass.csv')))
hdr = None
keep = []
for r in rows:
    if r and r[0] == 'Address':
        hdr = r
        keep.append(r)
    elif hdr and len(r) == len(hdr):
        keep.append(r)
# keep only rows with nonzero stall samples to bound the size
ws = hdr.index('Warp Stall Sampling (All Samples)') if hdr else None
out = [keep[0]] + [r for r in keep[1:] if ws is not None and r[ws] not in ('', '0')]
csv.writer(open('gpurun_out/r02_resident_sass_hot.csv', 'w')).writerows(out)
print(len(keep), len(out))
PY
ls -la $O
