# ncu --set full of one config-3 COLLAB call for each given lib
for l in "$@"; do
  n=$(basename $l .so)
  timeout 600 ncu --set full --clock-control none -k regex:ctf_ -s 2 -c 2 -o gpurun_out/prof_c3_$n python scripts/time_config3.py $l > /dev/null 2>&1
done
