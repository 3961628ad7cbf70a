# direct-path finish kernel variants: parity subset + cfg3 timing (PF on / off) against the HEAD library
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "direct or conventional or als or wide or paper or clamp or smoke" > gpurun_out/pf_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/pf_tests.log
for pf in 1 0; do FKK_DIRECT_PREFETCH=$pf timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn | tail -1 | sed "s/^/PF=$pf /"; done
FKK_LIB=$PWD/paper_2005_07132_b200/lib/libfkk_head.so timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn | tail -1 | sed "s/^/HEAD /"
