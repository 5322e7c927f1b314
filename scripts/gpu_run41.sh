for wm in 1 2; do echo "== wm $wm"; PMG_FD_WM=$wm timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior L[567]|wall"; done
for wm in 1 2; do echo "== c4 wm $wm"; PMG_FD_WM=$wm timeout 600 python scripts/breakdown.py c4 2 2>&1 | grep -E "fd_interior L[45]|wall"; done
