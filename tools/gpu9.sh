./tools/ubench/lat
python tools/timeline.py C2 40 | head -3
