python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -4
