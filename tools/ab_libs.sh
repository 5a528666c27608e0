# A/B of library builds: bash tools/ab_libs.sh libA.so libB.so ... (each run twice, interleaved):
# configs[3] bench (device-timed sweeps) and configs[0] on the resident stepper
for lib in "$@" "$@"; do
  PCGPU_LIB=$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-supp --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', 'cfg3', round(d['ms_per_step'],3), {k: round(v,4) for k,v in r['other_sweep_ms_per_launch'].items()})"
  PCGPU_LIB=$lib python tools/res_prof_cfg0.py | sed "s|^|$lib |"
done
