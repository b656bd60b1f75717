# Isolation probe: one table vs all tables per codec (product build), then the
# EMBC_DEBUG timelines of single-table huffman / vlz / raw decodes.
TAG=${1:-iso}
mkdir -p gpurun_out
(for T in 1 4 26; do timeout 300 python tools/probe_codec.py kg raw vlz huffman --tables $T; done) > gpurun_out/${TAG}_probe.log 2>&1
make -s -C paper_2407_04272_b200/csrc clean
make -s -j8 -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > /dev/null 2>&1
(for M in huffman vlz raw; do echo "== kg $M T=1"; timeout 300 python tools/probe_codec.py kg $M --tables 1; done) 2>&1 | grep -v KSPAN > gpurun_out/${TAG}_timeline.log
make -s -C paper_2407_04272_b200/csrc clean
cat gpurun_out/${TAG}_probe.log
grep -E "==|D1 " gpurun_out/${TAG}_timeline.log | tail -40
