for i in 1 2; do for l in ${LIBS:-default}; do
 if [ $l = default ]; then unset CHUNKLAB_LIB; else export CHUNKLAB_LIB=$l; fi
 echo -n "$l "; python tools/profile_token.py 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().split(' raw')[0]); print(d['minmax'], d['histogram'], d['one_call'])"
done; done
