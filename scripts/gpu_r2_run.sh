O=gpurun_out/m9
mkdir -p $O
timeout 900 python -m pytest tests/test_corpus.py tests/test_golden.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > $O/pytest_corpus.txt
cat $O/pytest_corpus.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
