# One GPU call: tests, bench line, ncu launch list, ncu full captures.
set -e; python paper_1209_3314_b200/build.py >/dev/null; python -c "import oracle; oracle.build()"; set +e
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile_engine -s 3 -c 1 -o gpurun_out/prof_tile python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > /dev/null 2>&1; echo "ncu tile rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:edt_rounds_raster -s 2 -c 1 -o gpurun_out/prof_edt_nuclei python scripts/prof_edt.py nuclei 4096 8 1 > /dev/null 2>&1; echo "ncu edt nuclei rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:edt_rounds_raster -s 2 -c 1 -o gpurun_out/prof_edt_blob python scripts/prof_edt.py blob 4096 8 1 > /dev/null 2>&1; echo "ncu edt blob rc=$?"
EDT_ENGINE=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:edt_block_kernel -s 2 -c 1 -o gpurun_out/prof_edtblock_nuclei python scripts/prof_edt.py nuclei 4096 8 1 > /dev/null 2>&1; echo "ncu edt block nuclei rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.json
DTYPE=2 ENGINE=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile_engine_reg32 -s 2 -c 1 -o gpurun_out/prof_reg32_i32 python scripts/prof_recon.py 4096 8 -1 0 rand 1 > /dev/null 2>&1; echo "ncu reg32 rc=$?"
