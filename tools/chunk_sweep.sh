mkdir -p gpurun_out
out=gpurun_out/chunk_sweep.txt
: > $out
for N in 100000; do for P in fp64 fp32; do
  for c in default 384 512 640 1024 1280 1536 2048; do
    if [ $c = default ]; then timeout 120 python tools/ab_env.py $N $P >> $out 2>&1
    else HAWKES_PAIRS_CHUNK=$c timeout 120 python tools/ab_env.py $N $P >> $out 2>&1; fi
  done; done; done
for N in 20000 50000; do
  for c in default 128 256 384 512; do
    if [ $c = default ]; then timeout 120 python tools/ab_env.py $N fp64 >> $out 2>&1
    else HAWKES_PAIRS_CHUNK=$c timeout 120 python tools/ab_env.py $N fp64 >> $out 2>&1; fi
  done; done
# repeat the default and best candidates for noise
for c in default 1024 1536; do
  if [ $c = default ]; then timeout 120 python tools/ab_env.py 100000 fp64 >> $out 2>&1
  else HAWKES_PAIRS_CHUNK=$c timeout 120 python tools/ab_env.py 100000 fp64 >> $out 2>&1; fi
done
cat $out
