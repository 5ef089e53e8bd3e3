python tools/timeline.py C2 40
python tools/timeline.py C2 1
