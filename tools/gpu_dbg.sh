# debug build (device counters/timestamps) + one TB bench, then the normal build again
mkdir -p gpurun_out
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > gpurun_out/dbg_build.log 2>&1
timeout 300 python bench.py --workload ${1:-tb} --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/dbg_run.log 2>&1
grep -v "^{" gpurun_out/dbg_run.log | tail -${2:-40}
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc >/dev/null 2>&1
