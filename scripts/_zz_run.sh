# c5 long-query solve A/B: cta2_solve variants (libs built into build_ab/ with -D flags)
# usage: bash scripts/_zz_run.sh label:lib:ctas_per_sm[:solve_kernel_pick] ...
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r label lib per_sm pick <<< "$spec"
  export SWMD_LIB=$lib SWMD_CTA_PER_SM=$per_sm SWMD_SOLVE_KERNEL=$pick
  [ -z "$SWMD_SOLVE_KERNEL" ] && unset SWMD_SOLVE_KERNEL
  [ -z "$SWMD_CTA_PER_SM" ] && unset SWMD_CTA_PER_SM
  timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fusion > gpurun_out/zz_$label.json 2> gpurun_out/zz_$label.err
  python -c "import json; d=json.loads(open('gpurun_out/zz_$label.json').read().strip().splitlines()[-1]); print('$label', 'solve ms', round(d['kernels']['solve_ms'],2))" || tail -3 gpurun_out/zz_$label.err
done
