mkdir -p gpurun_out
for fam in cholesky lu qr; do
  python bench.py --family $fam --steps 3 --warmup 3 --no-cpu-baseline --timings timings/b200_nb1024_ib128_tput.csv > gpurun_out/bench_${fam}_tput.json 2> /dev/null
done
