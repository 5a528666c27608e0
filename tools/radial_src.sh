# ncu source-level instruction counts of one cfg3 radial line launch
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-supp --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_line_exact_ws -s 14 -c 1 -o /tmp/rad $B > gpurun_out/ncu_rad.log 2>&1
ncu -i /tmp/rad.ncu-rep --page source --csv --print-source cuda > /tmp/rad_src.csv 2>&1
ncu -i /tmp/rad.ncu-rep --page source --csv --print-source sass > /tmp/rad_sass.csv 2>&1
python - <<'PY'
import csv
def keep(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None; res = []
    for r in rows:
        if r and r[0] in ('Line No', 'Address'):
            hdr = r; res.append(r); continue
        if r and r[0] == 'File Name':
            res.append(r); continue
        if hdr and len(r) == len(hdr):
            ie = hdr.index('Instructions Executed') if 'Instructions Executed' in hdr else None
            if ie is not None and r[ie] not in ('', '0'):
                res.append(r)
    csv.writer(open(out, 'w')).writerows(res)
    print(out, len(res))
keep('/tmp/rad_src.csv', 'gpurun_out/rad_src_hot.csv')
keep('/tmp/rad_sass.csv', 'gpurun_out/rad_sass_hot.csv')
PY
