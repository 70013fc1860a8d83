#!/bin/bash
# ncu --set full of the hot kernels: c2 reg_solve + cost_tmap (bench c2), c4 reg_solve<float>
# (one batch), c5 cta_solve; reports in gpurun_out/prof_<tag>.ncu-rep
mkdir -p gpurun_out
run() {  # tag, kernel regex, skip, count, command...
  tag=$1; rx=$2; sk=$3; cnt=$4; shift 4
  timeout 900 "$@" > gpurun_out/plain_$tag.log 2>&1 || { echo "$tag plain run failed"; return; }
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $cnt \
      -o gpurun_out/prof_$tag -f "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu_${tag}_rc=$?"
  python scripts/ncu_summary.py gpurun_out/prof_$tag.ncu-rep gpurun_out/ncu_$tag.json "$tag: $*" > /dev/null 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$tag.csv 2>/dev/null
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/ncu_src_$tag.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/prof_$tag.ncu-rep
  gzip -f gpurun_out/ncu_src_$tag.csv gpurun_out/ncu_raw_$tag.csv
}
for t in ${TAGS:-c2 c4 c5}; do
  case $t in
    c2) run c2 "reg_solve|cost_tmap" 4 2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c3 --no-fusion ;;
    c4) run c4 "reg_solve|gram32" 0 4 python bench.py --config c4 --steps 1 --warmup 3 ;;
    c5) run c5 "cta_solve|cost_tmap" 8 2 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-fusion ;;
    c3) run c3 "reg_solve|cost_tmap" 2 2 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-fusion ;;
  esac
done
