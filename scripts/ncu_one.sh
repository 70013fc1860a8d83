#!/bin/bash
# ncu --set full of one kernel launch: scripts/ncu_one.sh <tag> <kernel-regex> <skip> <command...>
# summary (scripts/ncu_summary.py) + gzipped raw/source csv in gpurun_out/, report deleted
tag=$1; rx=$2; sk=$3; shift 3
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c 1 \
    -o gpurun_out/prof_$tag -f "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_${tag}_rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_$tag.ncu-rep gpurun_out/ncu_$tag.json "$tag: $*" > /dev/null 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_raw_$tag.csv.gz
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/ncu_src_$tag.csv.gz
rm -f gpurun_out/prof_$tag.ncu-rep
