set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
for i in 1 2 3; do
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -rf --tb=line 2>&1 | grep -v "^\.\.\.\.\.\." | tail -8
done
