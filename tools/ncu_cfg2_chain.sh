python tools/cfg2_host_steps.py > gpurun_out/cfg2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_line_exact_ws8 -s 3 -c 1 -o /tmp/c2 python tools/cfg2_host_steps.py > gpurun_out/ncu_c2.log 2>&1
python tools/ncu_summary.py /tmp/c2.ncu-rep > gpurun_out/c2_ncu.txt 2>&1
ncu -i /tmp/c2.ncu-rep --page source --csv --print-source sass > /tmp/c2_sass.csv 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/c2_sass.csv')))
hdr = None; res = []
for r in rows:
    if r and r[0] == 'Address':
        hdr = r; res.append(r); continue
    if hdr and len(r) == len(hdr) and r[0].startswith('0x'):
        ie = hdr.index('Instructions Executed')
        if r[ie] not in ('', '0'):
            res.append(r)
csv.writer(open('gpurun_out/c2_sass_hot.csv', 'w')).writerows(res)
print(len(res))
PY
