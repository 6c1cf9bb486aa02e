for nt in 32768 16384 4096; do
  echo "nt=$nt new:"; SQR_PROBE_NT=$nt python tools/kernel_probe.py sample_qrcp 5
  echo "nt=$nt head:"; SQR_LIB=libsqr_head.so SQR_PROBE_NT=$nt python tools/kernel_probe.py sample_qrcp 5
done
