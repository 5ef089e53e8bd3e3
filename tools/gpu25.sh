for f in 2 2050 4098; do echo "== flags $f"; BQG_DEBUG_FLAGS=$f python tools/timeline.py C2 40 | grep -E "d query|d barrier|d reduce"; done
