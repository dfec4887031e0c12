REPS=2 compute-sanitizer --tool racecheck python scripts/debug_tiny.py 2>&1 | tail -6
bash scripts/sanitize.sh
