for lib in "" /root/repo/_variants/v_ns3.so /root/repo/_variants/v_ns4.so; do
  for c in c5 c3 c2; do if [ -n "$lib" ]; then export NGD_LIB_PATH=$lib; fi; timeout 300 python tools/matvec_one.py $c 3 2>&1 | tail -1 | sed "s|^|[$lib] |"; done
done
