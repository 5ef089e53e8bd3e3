BQG_DEBUG_FLAGS=114 python tools/timeline.py C2 1 | grep -E "build |rebuild|query "
