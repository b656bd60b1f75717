timeout 600 python -m pytest tests -q -m gpu -x --timeout 120 2>&1 | tail -2
for WL in kg tb sc; do timeout 300 python tools/probe_codec.py $WL prof 2>&1 | tail -1; done
