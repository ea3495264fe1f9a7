#!/bin/bash
# A/B timing of library variants: scripts/ab.sh variants/lib_x.so [more...]
# (default build vs each variant, alternating, two rounds)
VARIANTS=("$@")
for rep in 1 2; do
  for v in default "${VARIANTS[@]}"; do
    if [ "$v" != default ]; then export IWPP_B200_LIB=$PWD/$v; else unset IWPP_B200_LIB; fi
    line="$v:"
    for spec in "0 8 rand" "0 4 rand" "2 8 rand"; do
      set -- $spec
      r=$(DTYPE=$1 ENGINE=0 python scripts/prof_recon.py 4096 $2 -1 0 $3 40 2>&1 | tail -1 | sed 's/.*median \([0-9.]*\) ms.*/\1/')
      line="$line dt$1c$2=$r"
    done
    r=$(DTYPE=4 ENGINE=0 python scripts/prof_recon.py 16384 8 -1 0 imfill 10 2>&1 | tail -1 | sed 's/.*median \([0-9.]*\) ms.*/\1/')
    echo "$line imfill16k=$r"
  done
done
unset IWPP_B200_LIB
