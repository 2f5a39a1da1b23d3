for shape in "64 16 96 4" "64 8 96 8"; do
  TAG=new python tools/mac_bench.py $shape
  TAG=old HEAR_B200_LIB=lib_ab/libhear_b200.so python tools/mac_bench.py $shape
done
