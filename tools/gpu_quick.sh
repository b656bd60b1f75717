# One build -> measure iteration: GPU tests, per-codec probes (product build),
# then the EMBC_DEBUG timelines.  usage: bash tools/gpu_quick.sh TAG [workloads...]
TAG=${1:-q}; shift
WLS=${@:-kg tb}
mkdir -p gpurun_out
# a hang shows up here in a minute instead of in every later step
if ! timeout 90 python tools/probe_codec.py kg prof > gpurun_out/${TAG}_probe0.log 2>&1; then
  echo "probe hung or failed"; cat gpurun_out/${TAG}_probe0.log | tail -5; exit 1
fi
timeout 900 python -m pytest tests -q -m gpu -x --timeout 120 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.log
(for WL in $WLS; do timeout 120 python tools/probe_codec.py $WL prof raw vlz huffman; done) > gpurun_out/${TAG}_probe.log 2>&1
(timeout 120 python tools/probe_codec.py kg vlz huffman --tables 1) >> gpurun_out/${TAG}_probe.log 2>&1
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
(for WL in $WLS; do echo "== $WL"; timeout 120 python tools/probe_codec.py $WL prof; done) 2>&1 | grep -v KSPAN > gpurun_out/${TAG}_timeline.log
make -s -C paper_2407_04272_b200/csrc clean
cat gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_probe.log
grep -E "==|D1 |k_stats:|k_emit:" gpurun_out/${TAG}_timeline.log | tail -40
if [ -n "$NCU" ]; then
  make -s -j8 -C paper_2407_04272_b200/csrc > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_dec_main --launch-skip 6 -c 1 -f \
    -o gpurun_out/${TAG}_ncu python tools/probe_codec.py kg huffman --tables 26 > /dev/null 2>&1
fi
