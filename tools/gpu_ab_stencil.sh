# A/B of two library builds on the config-5 / config-3 field stencils (tools/probe_stencil2.py), then the
# per-tag breakdown of configs 3 and 5 on the current build
timeout 600 python tools/probe_stencil2.py paper_2305_19013_b200/libekcg_old.so 2>&1 | tail -4
timeout 600 python tools/probe_stencil2.py paper_2305_19013_b200/libekcg_b200.so 2>&1 | tail -4
timeout 600 python tools/breakdown.py --config 3 --kmax 60 2>&1 | tail -1
timeout 900 python tools/breakdown.py --config 5 --kmax 8 2>&1 | tail -1
