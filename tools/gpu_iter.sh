# One build -> measure iteration on the GPU box: GPU tests, per-codec probes,
# then the EMBC_DEBUG timeline build.  usage: bash tools/gpu_iter.sh TAG [probe args...]
TAG=${1:-it}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest.log
(for WL in kg tb; do timeout 300 python tools/probe_codec.py $WL prof raw vlz huffman; done) > gpurun_out/${TAG}_probe.log 2>&1
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
(for WL in kg tb; do timeout 300 python tools/probe_codec.py $WL prof; done) 2>&1 | grep -v KSPAN > gpurun_out/${TAG}_timeline.log
cat gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_probe.log
grep -E "D1 (vlzseg|hufblk|copy|finish|chunk)|k_stats:|k_emit:" gpurun_out/${TAG}_timeline.log | tail -14
