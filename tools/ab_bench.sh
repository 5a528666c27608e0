# A/B of library builds on the bench workload (device-timed per-launch sweep times).
# Variant builds: make -C paper_1912_03744_b200/csrc VARIANT=name EXTRA="-DX" -> _lib/ab/name/
for lib in paper_1912_03744_b200/_lib/libpcgpu.so paper_1912_03744_b200/_lib/ab/*/libpcgpu.so paper_1912_03744_b200/_lib/libpcgpu.so; do
  PCGPU_LIB=$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-supp --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', round(d['ms_per_step'],3), {k: round(v,4) for k,v in r['other_sweep_ms_per_launch'].items()})"
done
