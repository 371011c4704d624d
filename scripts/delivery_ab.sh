# acceptance criterion 5's replay alone: reference vs drop-in under each host wait policy
cd oracle/_ref/dropin
timeout 400 ./bench_read_ref delivery | sed 's/^{/{"arm": "ref", /'
for p in default spin yield blocking; do
  if [ $p = default ]; then timeout 400 ./bench_read_b200 delivery | sed 's/^{/{"arm": "b200", "sync": "default", /'
  else XPIR_SYNC=$p timeout 400 ./bench_read_b200 delivery | sed "s/^{/{\"arm\": \"b200\", \"sync\": \"$p\", /"; fi
done
