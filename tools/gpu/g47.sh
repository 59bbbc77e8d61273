python -m pytest tests -m gpu -q -s -k "config5" 2>&1 | grep -E "parity|passed|failed|Error" | head
