#!/bin/bash
# Round-2 re-captures after the EDT init changes (round 0 in the init, planar
# keys) and the banded recon queue order: same format as prof_r02.sh.
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
ATOM=lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
full() {
  timeout 900 ncu --set full --metrics $ATOM --clock-control none --import-source on \
    -k "regex:$2" -s $3 -c $3 -o $OUT/$1 python scripts/prof_r02.py $1 > $OUT/$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  python scripts/ncu_inst_lines.py $OUT/$1.ncu-rep 40 > $OUT/$1.lines.txt 2>/dev/null
  python scripts/ncu_sass_stalls.py $OUT/$1.ncu-rep 20 > $OUT/$1.sass.txt 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
full recon_u8_64k 'tile_engine_reg_kernel' 1
full edt_blob4k 'edt_rounds_raster_kernel|edt_init_key_rows_kernel|edt_finalize_key_kernel' 3
full edt_nuclei4k 'edt_rounds_raster_kernel|edt_init_key_rows_kernel|edt_finalize_key_kernel' 3
full edt_nuclei64k 'edt_init_key_rows_kernel|edt_finalize_key_kernel' 2
full edt_mg_blob4k 'mg_rounds_kernel' 1
du -sh $OUT
