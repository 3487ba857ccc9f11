for v in ${VARIANTS}; do env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python tools/time_generic.py 2>&1 | tail -1; done
