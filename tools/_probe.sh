bash tools/ab_libs.sh 3 5 _ab/minb9 _ab/minb10
