set -e; python paper_1209_3314_b200/build.py >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_edt.py -x -q 2>&1 | tail -3
python scripts/prof_edt.py blob 4096 8; python scripts/prof_edt.py nuclei 4096 8; python scripts/prof_edt.py blob 4096 4
ncu --set full --import-source on --clock-control none -k regex:edt_rounds -c 1 -o gpurun_out/edt_blob2 python scripts/prof_edt.py blob 4096 8 1 > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
