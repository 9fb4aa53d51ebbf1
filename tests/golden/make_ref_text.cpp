// Golden fixture: the REFERENCE library's own text writer on a VQH1 input.
// Reads argv[1] (VQH1, written by make_ref_text.py) with vqhull::read_points
// and writes argv[2] with vqhull::write_points(FileFormat::Text)
// (proj/src/io.cpp:100-121).  Built against oracle/_ref/libvqhull_ref.so and
// the reference headers by make_ref_text.py; runs only in the build container.
#include <cstdio>
#include <exception>
#include "vqhull/io.hpp"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    try {
        const vqhull::PointSet p = vqhull::read_points(argv[1]);
        vqhull::write_points(p, argv[2], vqhull::FileFormat::Text);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
