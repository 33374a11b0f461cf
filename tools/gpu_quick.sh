# quick GPU check: parity tests + C4 run timing + C2 timing
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/probe_iter.py point_to_plane ${1:-8} 2>&1 | grep -v "^pose"
python tools/c2_rep.py
