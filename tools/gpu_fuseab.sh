for f in "cholinv,vec,xr" "" "vec" "cholinv,vec" "vec,xr"; do echo "FUSE=$f"; FUSE=$f timeout 300 python tools/iter_profile.py 2 2>&1 | grep -E "^rep (1|2)"; done
