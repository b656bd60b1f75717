# Per-codec throughput probes, then the EMBC_DEBUG timeline build on the same workloads.
TAG=${1:-probe}
mkdir -p gpurun_out
for WL in kg tb sc; do timeout 600 python tools/probe_codec.py $WL; done > gpurun_out/${TAG}_codec.log 2>&1
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
for WL in kg tb; do timeout 600 python tools/probe_codec.py $WL prof; done > gpurun_out/${TAG}_timeline.log 2>&1
cat gpurun_out/${TAG}_codec.log
