# Round-2 final evidence on the B200 (through gpurun): the default bench line,
# the reference arm, the launch list, ncu --set full of one radial and one
# axial line launch (summarised on the box), and the resident timings.
set -x
O=gpurun_out
python bench.py > $O/bench_final.json 2> $O/bench_final.err
python bench.py --impl reference > $O/bench_reference_final.json 2> $O/bench_reference_final.err
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-supp --no-e2e"
$B > $O/plain_final.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_final.csv $B > $O/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_exact_ws -s 14 -c 2 -o /tmp/fin_ws $B > $O/ncu_ws.log 2>&1
python tools/ncu_summary.py /tmp/fin_ws.ncu-rep > $O/final_ws_ncu.txt 2>&1
python tools/res_timing.py --configs cfg0,paper,cfg2,cfg4 > $O/res_timing_final.json 2>&1
ls -la $O
