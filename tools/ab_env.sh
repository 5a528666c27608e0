# A/B of environment switches on the bench workload (device-timed per-launch sweep times)
for env in "X=1" "PCGPU_NO_K4FUSE=1" "X=1" "PCGPU_NO_K4FUSE=1"; do
  env $env python bench.py --steps 10 --warmup 3 --no-cpu --no-supp --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$env', round(d['ms_per_step'],3), d['value'], {k: round(v,4) for k,v in r['other_sweep_ms_per_launch'].items()})"
done
