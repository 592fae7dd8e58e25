# the reference's bundled part (proj/src/splines.cpp:408-438)
[geometry]
case = quarter_cylinder
