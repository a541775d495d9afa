mkdir -p gpurun_out
python scripts/pcie_probe.py > gpurun_out/e2e_diag.log 2>&1
NB=0 python scripts/e2e_probe.py >> gpurun_out/e2e_diag.log 2>&1
NB=1 python scripts/e2e_probe.py >> gpurun_out/e2e_diag.log 2>&1
NB=1 NFFT45_STREAM_CHUNK=128 python scripts/e2e_probe.py >> gpurun_out/e2e_diag.log 2>&1
nvidia-smi topo -m >> gpurun_out/e2e_diag.log 2>&1
lscpu | head -20 >> gpurun_out/e2e_diag.log
cat gpurun_out/e2e_diag.log
