# Round-2 profile capture on the B200 (run through gpurun): the bench line, the
# launch list, and ncu --set full of the top kernels summarised as text on the
# box (the .ncu-rep files are too large to bring back).
set -x
O=gpurun_out
python bench.py --steps 10 --warmup 3 > $O/bench_r02.json 2> $O/bench_r02.err
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-supp --no-e2e"
$B > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/r02_launches.csv $B > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_exact_ws -s 14 -c 2 -o /tmp/r02_ws $B > $O/ncu2.log 2>&1
python tools/ncu_summary.py /tmp/r02_ws.ncu-rep > $O/r02_ws_ncu.txt 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_explicit_axial_t3|k_axial_rhs_t3" -s 4 -c 2 -o /tmp/r02_k34 $B > $O/ncu3.log 2>&1
python tools/ncu_summary.py /tmp/r02_k34.ncu-rep > $O/r02_k34_ncu.txt 2>&1
R="python tools/res_profile_run.py"
$R > $O/plain_res.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o /tmp/r02_res $R > $O/ncu4.log 2>&1
python tools/ncu_summary.py /tmp/r02_res.ncu-rep > $O/r02_resident_ncu.txt 2>&1
ncu -i /tmp/r02_res.ncu-rep --page source --csv --print-source cuda > $O/r02_resident_src.csv 2>&1
ls -la $O
