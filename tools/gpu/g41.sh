python -m pytest tests -m gpu -q -x -k "graph_cache or repeated" 2>&1 | tail -3
