# e2e (batch) under fetch knobs: wire chunks and host threads
for cfg in "SSB_WIRE_CHUNKS=64" "SSB_WIRE_CHUNKS=128" "SSB_WIRE_CHUNKS=256" "SSB_WIRE_CHUNKS=32" "SSB_HOST_THREADS=12" "SSB_HOST_THREADS=15" "SSB_WIRE_CHUNKS=64"; do
  echo "== $cfg $(env $cfg python scripts/sweep_wire_direct.py 32 2>&1 | head -1)"
done
