for lib in "$@"; do timeout 300 python tools/kbench.py $lib 4096 2>&1 | tail -1; done
for lib in "$@"; do timeout 300 python tools/kbench.py $lib 4096 2>&1 | tail -1; done
