# Fig. 3 methodology on B200: fft_pad vs tft device ns per product of one
# batched call (scripts/fig3_device.py): just past each power of two 2048 ..
# 32768, and whole octaves (n in (L/2, L]) for the staircase against the
# truncated engine, with p2 (Harvey ranges) and p3 (canonical).
mkdir -p gpurun_out/sweep
S="python scripts/fig3_device.py --reps ${REPS:-15}"
$S --min 1900 --max 2300 --step 8 -o gpurun_out/sweep/sweep_fig3_2048.csv
$S --min 4000 --max 4600 --step 12 -o gpurun_out/sweep/sweep_fig3_4096.csv
$S --min 8100 --max 9200 --step 20 -o gpurun_out/sweep/sweep_fig3_8192.csv
$S --min 16300 --max 18500 --step 44 -o gpurun_out/sweep/sweep_fig3_16384.csv
$S --min 32500 --max 37000 --step 180 -o gpurun_out/sweep/sweep_fig3_32768.csv
$S --min 520 --max 1024 --step 8 -o gpurun_out/sweep/octave_1024.csv
$S --min 1032 --max 2048 --step 16 -o gpurun_out/sweep/octave_2048.csv
$S --min 2056 --max 4096 --step 40 -o gpurun_out/sweep/octave_4096.csv
$S --prime 2013265921 --min 2056 --max 4096 --step 40 -o gpurun_out/sweep/octave_4096_p3.csv
$S --min 4112 --max 8192 --step 80 -o gpurun_out/sweep/octave_8192.csv
$S --min 16448 --max 32768 --step 320 -o gpurun_out/sweep/octave_32768.csv
python scripts/sweep_summary.py gpurun_out/sweep/*.csv | grep -E "csv|worst"
