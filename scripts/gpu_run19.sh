for mk in 160 16; do echo "STREAMK_MIN_KB=$mk"; ENERGON_STREAMK_MIN_KB=$mk TPS=1,2,4,8 timeout 500 python scripts/sweep_tiles.py 2>&1 | head -16 | python -c "
import sys,re
for l in sys.stdin:
    m=re.match(r'(tp\d \w+) .*?\'1256\': (\d+).*\'cublas\': (\d+)', l)
    if m: print(m.group(1), m.group(2), 'cublas', m.group(3))"; done
