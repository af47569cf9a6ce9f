for ch in 2 3 4 6 8 16; do
  echo "== chunks $ch"
  MC_STREAM_IN_MIN_MB=0 MC_STREAM_IN_CHUNKS=$ch python scripts/zc_tma_probe.py 2>&1 | grep "zero copy"
done
echo "== default (zero copy)"; python scripts/zc_tma_probe.py 2>&1 | grep "zero copy"
