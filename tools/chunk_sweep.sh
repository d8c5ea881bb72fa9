for c in 3 4 5 6 7 8 10 12; do
  echo "nchunk=$c"; STB_NCHUNK=$c python tools/order_sweep.py 8 4 2>&1 | grep so=
done
