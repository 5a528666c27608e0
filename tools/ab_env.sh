# A/B of environment switches on the bench workload (device-timed per-launch sweep times)
# usage: bash tools/ab_env.sh "X=1" "PCGPU_FLOW=0" ...   (each env pair runs twice, interleaved)
for env in "$@" "$@"; do
  env $env python bench.py --steps 10 --warmup 3 --no-cpu --no-supp --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$env', round(d['ms_per_step'],3), '%.4g' % d['value'], {k: round(v,4) for k,v in r['other_sweep_ms_per_launch'].items()}, d['config']['picard'])"
done
