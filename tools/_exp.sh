for v in R7 KI1 KI1R7; do
  KNNM_LIB=$PWD/tools/_var/libknnm_$v.so timeout 300 python tools/_exp.py c3 0.3 1 2>&1 | tail -1
done
