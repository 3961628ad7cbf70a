for b in 131072 262144 360000 703040; do echo "batch=$b"; FKK_DIRECT_BATCH=$b timeout 300 python tools/prof_direct.py 703026 2 2>&1 | grep -v Warn | tail -1; done
