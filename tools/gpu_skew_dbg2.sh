for sh in "32 256 256" "256 8 256" "128 256 256" "256 256 256"; do echo "shape $sh"; CF_DIC_DEBUG=1 timeout 300 python tools/skew_one.py $sh 1 2>&1 | grep -E "late|iterations" | tail -2; done
