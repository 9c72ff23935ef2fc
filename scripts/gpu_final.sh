# final check of HEAD: GPU suite, smoke, default bench line, reference arm
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>/dev/null | cut -c1-400
timeout 600 python bench.py --impl reference 2>/dev/null | cut -c1-300
