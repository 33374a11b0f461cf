# A/B of engine variants (tools/variants.sh): C4 run both metrics, C4 iterate at identity, C2 query, C5 2^22 iterate
for v in "$@"; do
  for m in point_to_plane point_to_point; do
    METRIC=$m PYTHONPATH=tools/ubench/var_$v python tools/time_c4_skin.py
  done
  PYTHONPATH=tools/ubench/var_$v python tools/time_engine.py
done
