/* oracle/shim/png.h — TEST INFRASTRUCTURE ONLY.
 *
 * libpng is a third-party dependency of the reference's image I/O
 * (`proj/src/image.cpp:9,92-169`) that is absent from this image. PNG I/O is out of
 * scope for the hot path. This stub declares the libpng symbols the
 * reference calls; png_create_{read,write}_struct return NULL, so every PNG
 * read/write in the oracle build throws the reference's own IoError
 * (`image.cpp:97-101,139-143`). PGM I/O is unaffected.
 */
#ifndef WBX_ORACLE_PNG_STUB_H
#define WBX_ORACLE_PNG_STUB_H

#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned int png_uint_32;
typedef struct wbx_png_struct_s* png_structp;
typedef struct wbx_png_info_s* png_infop;
typedef unsigned char* png_bytep;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_MASK_COLOR 2
#define PNG_COLOR_MASK_ALPHA 4
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

static jmp_buf wbx_png_stub_jmp;
#define png_jmpbuf(p) (((void)(p)), wbx_png_stub_jmp)

static inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_infop png_create_info_struct(png_structp) { return NULL; }
static inline void png_destroy_read_struct(png_structp*, png_infop*, png_infop*) {}
static inline void png_destroy_write_struct(png_structp*, png_infop*) {}
static inline void png_init_io(png_structp, FILE*) {}
static inline void png_read_info(png_structp, png_infop) {}
static inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
static inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
static inline int png_get_bit_depth(png_structp, png_infop) { return 8; }
static inline int png_get_color_type(png_structp, png_infop) { return 0; }
static inline void png_set_palette_to_rgb(png_structp) {}
static inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
static inline void png_set_rgb_to_gray(png_structp, int, double, double) {}
static inline void png_set_strip_alpha(png_structp) {}
static inline void png_read_update_info(png_structp, png_infop) {}
static inline size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
static inline void png_read_row(png_structp, png_bytep, png_bytep) {}
static inline void png_read_end(png_structp, png_infop) {}
static inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int,
                                int, int) {}
static inline void png_write_info(png_structp, png_infop) {}
static inline void png_write_row(png_structp, png_bytep) {}
static inline void png_write_end(png_structp, png_infop) {}

#ifdef __cplusplus
}
#endif

#endif
