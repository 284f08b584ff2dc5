timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -8
./build/dropin_check 0 2>&1 | tail -14
