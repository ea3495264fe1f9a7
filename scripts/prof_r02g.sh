#!/bin/bash
# Round-2 (session 5) re-captures final build of the session (binary engine, event-free timed step, 8-conn cooperative EDT compaction): both bench
# arms, the launch list of the headline bench command and one `--set full`
# capture of the imfill kernels (same format as prof_r02.sh; summarised by
# `scripts/summarize_r02.py gpurun_out/r02g r02g`).
set -u
OUT=gpurun_out/r02g
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
if [ $# -gt 0 ]; then  # only the named cases: prof_r02c.sh CASE REGEX COUNT
  full "$1" "$2" "$3"; exit 0
fi
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu > $OUT/launches.log 2>&1
echo "launches rc=$?"
full imfill_16k 'tile_engine_bin_kernel|bin_pack_kernel|bin_unpack_kernel' 3
full edt_blob4k 'edt_rounds_raster_kernel' 1
du -sh $OUT
