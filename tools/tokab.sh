for i in 1 2; do for l in build/variants/h16.so build/variants/h24.so build/variants/h32.so; do
 if [ $l = default ]; then unset CHUNKLAB_LIB; else export CHUNKLAB_LIB=$l; fi
 echo -n "$l "; python tools/profile_token.py 2>&1 | tail -1 | cut -c1-110
done; done
