for lib in build/liblsk_base.so build/liblsk_prul8.so build/liblsk_prul10.so build/liblsk_base.so; do
  echo "$lib c4 $(LSK_LIB=$lib timeout 300 python tools/profile_points.py c4 --iters 20 2>&1 | tail -1)"
  echo "$lib c5 $(LSK_LIB=$lib timeout 300 python tools/profile_points.py c5 --iters 200 2>&1 | tail -1)"
done
