for C in 0 256 512 2048; do
  echo "cper=$C $(EMBC_CPER=$C timeout 300 python tools/probe_codec.py sc prof 2>&1 | tail -1)"
done
