timeout 600 python -m pytest tests -m gpu -x -q -k "transforms or mips" 2>&1 | tail -25
