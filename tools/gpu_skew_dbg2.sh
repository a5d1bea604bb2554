for sh in "32 16 256" "128 4 256"; do echo "shape $sh"; CF_DIC_DEBUG=1 timeout 300 python tools/skew_one.py $sh 1 2>&1 | tail -6; done
