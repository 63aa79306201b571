for v in libngd_b200.so _var_s1.so _var_s3.so; do
  echo "== $v"
  NGD_LIB_PATH=paper_2505_11638_b200/$v python tools/sketch_one.py c5
  NGD_LIB_PATH=paper_2505_11638_b200/$v python tools/matvec_one.py c5 3
  NGD_LIB_PATH=paper_2505_11638_b200/$v python tools/sketch_one.py c2
done
