# A/B of the certified warm-start variants (tools/variants.sh) on C4, both metrics
for v in "$@"; do
  for m in point_to_plane point_to_point; do
    METRIC=$m GRID="${GRID:-0.001,0.005,16}" PYTHONPATH=tools/ubench/var_$v python tools/time_c4_skin.py
  done
done
