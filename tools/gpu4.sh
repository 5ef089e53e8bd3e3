python tools/timeline.py C2
python tools/timeline.py C1
python tools/timeline.py C3
