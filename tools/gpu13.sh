for f in 18 50; do echo "== flags $f"; BQG_DEBUG_FLAGS=$f python tools/timeline.py C2 40 | grep -E "build |query "; done
for f in 18 50; do echo "== flags $f 1copy"; BQG_DEBUG_FLAGS=$f python tools/timeline.py C2 1 | grep -E "build |query "; done
