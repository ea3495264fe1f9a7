set -e; python paper_1209_3314_b200/build.py >/dev/null; set +e
ncu --set full --import-source on --clock-control none -k regex:tile_engine -s 2 -c 1 -o gpurun_out/tile_w1 python scripts/prof_recon.py 4096 8 1 0 rand 1 > gpurun_out/ncu1.log 2>&1
tail -1 gpurun_out/ncu1.log
