# ncu of the 9-bucket quad kernel and the quad kernel at B = 8192 (second launch of each); N from $1
N=${1:-262144}
for k in 10 8; do
  name=$([ $k = 10 ] && echo k_scan_m4rm_q9 || echo k_scan_m4rm_q)
  timeout 900 ncu --set full --clock-control none --import-source on -k "$name" --launch-skip 1 -c 1 \
    -o gpurun_out/q9_k${k}_n$N python scripts/one_scan.py $k $N 4096 8192 2 > gpurun_out/prof_q9_k${k}_n$N.log 2>&1
  tail -2 gpurun_out/prof_q9_k${k}_n$N.log
done
