T=1758 H=768 TPS=1 timeout 300 python scripts/sweep_tiles.py 2>&1 | head -4
T=4096 H=768 TPS=1 timeout 300 python scripts/sweep_tiles.py 2>&1 | head -4
