for p in 0 1 2 0 1; do echo "PDL=$p"; PDL=$p timeout 300 python tools/iter_profile.py 2 2>&1 | grep -E "^rep (1|2)"; done
PDL=1 timeout 300 python tools/iter_profile.py 3 2>&1 | grep -E "^rep (1|2)" | head -1
