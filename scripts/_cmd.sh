timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python scripts/e2e_breakdown.py c2
