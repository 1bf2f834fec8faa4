out=gpurun_out/j2
mkdir -p $out
python tools/j2_once.py 10 > $out/once.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_face_stencil -s 1 -c 1 -o $out/j2 python tools/j2_once.py 10 > $out/ncu.log 2>&1
ncu -i $out/j2.ncu-rep --page details --csv > $out/details.csv 2>/dev/null
ncu -i $out/j2.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
rm -f $out/j2.ncu-rep
