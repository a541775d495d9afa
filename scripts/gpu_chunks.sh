mkdir -p gpurun_out
for c in 64 128 256 512; do NB=1 NFFT45_STREAM_CHUNK=$c python scripts/e2e_probe.py; done > gpurun_out/chunks.log 2>&1
cat gpurun_out/chunks.log
