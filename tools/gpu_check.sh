set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -20
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -40
