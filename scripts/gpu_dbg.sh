python scripts/debug_tiny.py
ENERGON_NO_PDL=1 python scripts/debug_tiny.py
REPS=2 compute-sanitizer --tool racecheck python scripts/debug_tiny.py 2>&1 | tail -8
