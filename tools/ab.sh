set -e
for i in 1 2; do
for c in 8 0; do CL_SCAN_CFG=$c python tools/profile_stages.py --reps 30 --median 2>&1 | grep cfg; done
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
