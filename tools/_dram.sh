ARGS="--M 16384 --T 512 --reps 1"
for mb in 128 64; do
timeout 300 python tools/prof_align.py $ARGS --work-mb $mb > /dev/null 2>&1 && \
timeout 600 ncu --replay-mode application --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"contract|fft" -s 60 -c 4 --csv python tools/prof_align.py $ARGS --work-mb $mb 2>/dev/null | grep -v "^==" | tail -13 > gpurun_out/dram_$mb.csv
echo "== $mb"; cat gpurun_out/dram_$mb.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | tail -12
done
