# where C2's end-to-end time goes (flush + sync as bench.py; re-costed points)
set -x
python scripts/e2e_probe.py c2 400
