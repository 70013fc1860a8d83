timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
TAG=tmap timeout 300 python scripts/cost_probe.py c2 c3 2>&1 | grep cost
