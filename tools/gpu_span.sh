# debug build: per-call kernel spans (globaltimer) of k_encode / k_dec_main, and the gaps between them
mkdir -p gpurun_out
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc EXTRA=-DEMBC_DEBUG > gpurun_out/dbg_build.log 2>&1
timeout 300 python bench.py --workload ${1:-kg} --no-cpu-baseline --steps 12 --warmup 3 > gpurun_out/span.log 2>&1
grep KSPAN gpurun_out/span.log | python -c "
import sys
ev=[l.split() for l in sys.stdin]
ev=sorted([(k, int(a), int(b)) for _, k, a, b in ev], key=lambda e: e[1])
for i, ((k0,a0,b0),(k1,a1,b1)) in enumerate(zip(ev, ev[1:])):
    print(f'{i:4d} {k0} {(b0-a0)/1e3:7.2f} us, gap to {k1} {(a1-b0)/1e3:8.2f} us')
" > gpurun_out/span_pairs.txt
make -s -C paper_2407_04272_b200/csrc clean >/dev/null; make -s -C paper_2407_04272_b200/csrc >/dev/null 2>&1
