# debug build (device timestamps) + kg and tb bench, then the normal build again
mkdir -p gpurun_out
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > gpurun_out/dbg_build.log 2>&1
for w in kg tb; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/dbg_run_$w.log 2>&1
echo "== $w"; grep -v "^{" gpurun_out/dbg_run_$w.log | tail -${1:-14}
done
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc >/dev/null 2>&1
