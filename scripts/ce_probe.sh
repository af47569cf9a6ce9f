python scripts/ce_enqueue_probe.py default zc in pipe
for k in 2 4 8 16; do MC_CE_CHUNKS=$k python scripts/ce_enqueue_probe.py ce; done
