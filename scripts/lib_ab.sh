# A/B of two library builds: LIBS="lib/libnfft45_old.so lib/libnfft45_new.so" CMD="python scripts/single_probe.py"
for l in $LIBS; do echo "== $l"; NFFT45_LIB=$PWD/paper_1604_06236_b200/$l $CMD; done
