for k in 4 8 16; do MC_STREAM_IN_CHUNKS=$k python scripts/ce_enqueue_probe.py in; done
python scripts/ce_enqueue_probe.py zc
