# Per-codec probes (product build), then the EMBC_DEBUG timeline build for each workload.
# usage: bash tools/gpu_timeline.sh TAG [workloads...]
TAG=${1:-tl}; shift
WLS=${@:-kg tb}
mkdir -p gpurun_out
(for WL in $WLS; do timeout 300 python tools/probe_codec.py $WL prof raw vlz huffman; done) > gpurun_out/${TAG}_probe.log 2>&1
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
(for WL in $WLS; do echo "== $WL"; timeout 300 python tools/probe_codec.py $WL prof; done) 2>&1 | grep -v KSPAN > gpurun_out/${TAG}_timeline.log
make -s -C paper_2407_04272_b200/csrc clean
cat gpurun_out/${TAG}_probe.log
grep -E "==|D1 |k_stats:|k_emit:|E[0-9]" gpurun_out/${TAG}_timeline.log | tail -60
