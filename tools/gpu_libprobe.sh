# probe_codec over the current tree and every tools/ablibs/lib_*.so (EMBC_LIB)
WLS=${@:-tb sc}
for WL in $WLS; do
  echo "cur $(timeout 300 python tools/probe_codec.py $WL prof 2>&1 | tail -1)"
  for L in tools/ablibs/lib_*.so; do echo "$(basename $L) $(EMBC_LIB=$PWD/$L timeout 300 python tools/probe_codec.py $WL prof 2>&1 | tail -1)"; done
done
