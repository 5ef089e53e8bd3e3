for f in 2 6 10; do echo "== flags $f"; BQG_DEBUG_FLAGS=$f python tools/timeline.py C2 | grep -E "query |fence|finalize|end "; done
