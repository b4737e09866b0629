for g in 74 111 148 222 296 444; do BCN_PACE_GRID=$g timeout 120 python tools/sustain.py --seconds 4 --only f64_fp64_paced7200 | sed "s/^{/{\"grid\": $g, /"; sleep 2; done
