for p in 1 0 1 0; do echo "PDL=$p"; PDL=$p timeout 300 python tools/iter_profile.py 2 2>&1 | grep -E "^rep (1|2)"; done
