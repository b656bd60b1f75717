# EMBC_DEBUG timelines only. usage: bash tools/gpu_tl.sh TAG [workloads...]
TAG=${1:-tl}; shift
WLS=${@:-kg tb}
mkdir -p gpurun_out
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
(for WL in $WLS; do echo "== $WL"; timeout 120 python tools/probe_codec.py $WL prof; done) 2>&1 | grep -v KSPAN > gpurun_out/${TAG}_timeline.log
make -s -C paper_2407_04272_b200/csrc clean
grep -E "==|D1 (vlzseg|hufblk|copy|finish|chunk)|^(kg|tb)" gpurun_out/${TAG}_timeline.log
