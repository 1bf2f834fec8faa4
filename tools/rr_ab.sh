# ncu launch durations of the restriction-fused residual (k_face_stencil<3>) on config 2 L10 and config 3 L9 / L8
for args in "cfg2 10" "cfg3 9" "cfg3 8"; do timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_face_stencil -c 3 python tools/rr_time.py $args 2 2>&1 | grep -E "gpu__time_duration" | tail -1; done
