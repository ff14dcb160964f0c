for v in lib acro5 acro4; do
  L=paper_2408_00930_b200/lib/libws.so; [ $v != lib ] && L=paper_2408_00930_b200/lib/$v/libws.so
  for E in 100000 400000; do WS_LIBWS=$L python tools/time_rollout.py acrobot $E 500 5 | sed "s/^/$v /"; done
  WS_LIBWS=$L python tools/time_rollout.py acrobot 100000 500 5 64 | sed "s/^/$v /"
done
