echo "== 1 copy"; python tools/timeline.py C2 1 | grep -E "build |query |fence|finalize|end "
echo "== 40 copies"; python tools/timeline.py C2 40 | grep -E "build |query |fence|finalize|end "
echo "== 40 copies, no loads in finalize"; BQG_DEBUG_FLAGS=10 python tools/timeline.py C2 40 | grep -E "build |query |fence|finalize|end "
