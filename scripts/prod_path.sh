# production-path measurements of the reference's own harness, both arms
cd oracle/_ref/dropin
OUT=../../../gpurun_out/prod_path.jsonl; : > $OUT
for arm in b200 ref; do
  timeout 900 ./bench_read_$arm process 10000,100000,1000000 20 | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
  timeout 600 ./bench_read_$arm concurrent 10000 64 16 | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
  timeout 600 ./bench_read_$arm concurrent 100000 64 8 | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
  timeout 600 ./bench_read_$arm writes 131072 500 8 | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
  timeout 600 ./bench_read_$arm writes 32768 64 16 | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
  timeout 400 ./bench_read_$arm delivery | sed "s/^{/{\"arm\": \"$arm\", /" >> $OUT
done
echo "host: $(nproc) cores, $(grep -m1 'model name' /proc/cpuinfo)" >> ../../../gpurun_out/prod_path_host.txt
timeout 1200 ./acceptance_b200 > ../../../gpurun_out/acceptance_b200.txt 2>&1
OBLOG_B200_HOST_SNAPSHOTS=1 timeout 1200 ./acceptance_b200 > ../../../gpurun_out/acceptance_b200_hostsnap.txt 2>&1
timeout 1200 ./acceptance_ref > ../../../gpurun_out/acceptance_ref.txt 2>&1
cat $OUT | cut -c1-200
grep CRITERION ../../../gpurun_out/acceptance_*.txt | cut -c1-160
