set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python tools/variant_bench.py
python tools/e2e_profile.py 2>&1 | tail -24
