#!/bin/bash
# ab_krows.sh OUTDIR FAMILIES VARIANT...  -- config-3 block-row kernel timings for the
# in-tree library ("new") and each paper_2505_13723_b200/_lib_VARIANT build
set -u
out=$1; fams=$2; shift 2
mkdir -p $out
for fam in $fams; do
  for lib in new "$@"; do
    if [ $lib = new ]; then unset SAP_LIB_PATH; else export SAP_LIB_PATH=$PWD/paper_2505_13723_b200/_lib_$lib/libsapgp_b200.so; fi
    timeout 120 python scripts/krows_once.py --family $fam --reps 12 >> $out/times.log 2>&1 && echo "  ^ $lib $fam" >> $out/times.log
  done
done
unset SAP_LIB_PATH
