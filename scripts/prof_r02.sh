#!/bin/bash
# Round-2 ncu evidence (run on the GPU box from the repo root):
#   launch list of the headline bench command + one `--set full` capture per
#   kernel family, with the L2 atomic counters added.
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
ATOM=lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
full() {  # case kernel-regex count
  timeout 900 ncu --set full --metrics $ATOM --clock-control none --import-source on \
    -k "regex:$2" -s $3 -c $3 -o $OUT/$1 python scripts/prof_r02.py $1 > $OUT/$1.log 2>&1
  echo "$1 rc=$?"
  # compact evidence only (gpurun_out travels back only under 64 MiB):
  # every metric of every captured launch, and the per-line stall summary
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  python scripts/ncu_inst_lines.py $OUT/$1.ncu-rep 40 > $OUT/$1.lines.txt 2>/dev/null
  python scripts/ncu_sass_stalls.py $OUT/$1.ncu-rep 20 > $OUT/$1.sass.txt 2>/dev/null
  [ "$1" = recon_u8_4k ] || rm -f $OUT/$1.ncu-rep
}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu > $OUT/launches.log 2>&1
echo "launches rc=$?"
full recon_u8_4k 'tile_engine_reg_kernel' 1
full recon_i32_4k 'tile_engine_reg32_kernel' 1
full recon_u8_64k 'tile_engine_reg_kernel' 1
full imfill_16k 'tile_engine_bin_kernel|bin_pack_kernel|bin_unpack_kernel' 3
full stages_16k 'row_sweep|col_|seed_scan|check_le' 6
full edt_blob4k 'edt_rounds_raster_kernel|edt_init_key_rows_kernel|edt_finalize_key_kernel' 3
full edt_nuclei4k 'edt_rounds_raster_kernel|edt_init_key_rows_kernel|edt_finalize_key_kernel' 3
full edt_mg_blob4k 'mg_rounds_kernel' 1
full edt_nuclei64k 'edt_init_key_rows_kernel|edt_finalize_key_kernel' 2
python scripts/probe_pcie.py > $OUT/pcie.txt 2>&1
ls -la $OUT; du -sh $OUT
