set -e; python paper_1209_3314_b200/build.py >/dev/null; set +e
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/prof_recon.py 4096 8 1 0 rand 5; python scripts/prof_recon.py 4096 4 1 0 rand 5
for h in 0 16; do HTH=$h python scripts/prof_recon.py 16384 4 1 0 imfill 3; HTH=$h python scripts/prof_recon.py 16384 8 1 0 imfill 3; done
