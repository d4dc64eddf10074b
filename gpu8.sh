python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
python tools/ncu_decode.py > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:decode_persistent -s 1 -c 1 \
    -o gpurun_out/pk_full_r1 python tools/ncu_decode.py > gpurun_out/ncu_run2.log 2>&1
echo full rc=$?
