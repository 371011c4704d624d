# kernel 8 (then the byte-table quad kernel) vs candidate 10 (the 9-bucket tables, now kernel 8) vs 5 on a 1 GiB store at the batch sizes the
# cost model routes to them
for S in 512 1024 4096 8192; do
  N=$(( (1 << 30) / S ))
  for B in 2048 4096 6144 8192 16384; do
    for k in 8 10 5; do python scripts/time_scan.py $k $N $S $B 3; done
  done
done
