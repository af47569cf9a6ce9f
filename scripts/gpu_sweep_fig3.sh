# Fig. 3 methodology on B200: fft_pad vs tft device ns per product of one
# batched call (scripts/fig3_device.py), across 2048 / 4096 / 8192 / 16384.
mkdir -p gpurun_out/sweep
S="python scripts/fig3_device.py --reps ${REPS:-15}"
$S --min 1900 --max 2300 --step 8 -o gpurun_out/sweep/sweep_fig3_2048.csv
$S --min 4000 --max 4600 --step 12 -o gpurun_out/sweep/sweep_fig3_4096.csv
$S --min 8100 --max 9200 --step 20 -o gpurun_out/sweep/sweep_fig3_8192.csv
$S --min 16300 --max 18500 --step 44 -o gpurun_out/sweep/sweep_fig3_16384.csv
python scripts/fig3_device.py --reps ${REPS:-15} --min 32500 --max 37000 --step 180 -o gpurun_out/sweep/sweep_fig3_32768.csv
python scripts/sweep_summary.py gpurun_out/sweep/sweep_fig3_*.csv
