cp paper_2001_08250_b200/libxpir.so /tmp/libxpir_orig.so
for ni in 1 2 3; do cp paper_2001_08250_b200/libxpir_ni$ni.so paper_2001_08250_b200/libxpir.so; echo NI=$ni; S=4096 python scripts/sweep_direct.py run; done
cp /tmp/libxpir_orig.so paper_2001_08250_b200/libxpir.so
